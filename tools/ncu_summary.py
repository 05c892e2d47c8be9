"""Summarise an `ncu --metrics ... --csv` launch list of one bench command into
profiles/ncu_summary.json (read by bench.py's roofline: `traffic` and the DMMA-pipe figure).

    python tools/ncu_summary.py <workload> <kernel regex> <ncu.csv> [source-name]

Per workload it records, over every captured launch of the dominant kernel: the mean DRAM
bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), the duration-weighted mean
DMMA-pipe and FP64-pipe utilisation, and the launch count.  ncu serialises and cold-starts
each launch, so these are per-launch hardware counters, not the bench's timing."""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")


def parse(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        rows.append(r)
    return rows


def scale(v, unit):
    v = float(v.replace(",", ""))
    u = (unit or "").lower()
    return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
                "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u, 1.0)


def main():
    wl, pat, path = sys.argv[1], sys.argv[2], sys.argv[3]
    src = sys.argv[4] if len(sys.argv) > 4 else os.path.relpath(path, ROOT)
    rows = [r for r in parse(path) if re.search(pat, r["Kernel Name"])]
    by = {}
    for r in rows:
        by.setdefault(r["ID"], {})[r["Metric Name"]] = scale(r["Metric Value"], r["Metric Unit"]) \
            if r["Metric Unit"] != "%" else float(r["Metric Value"])
    launches = list(by.values())
    n = len(launches)
    t = [m.get("gpu__time_duration.sum", 0.0) for m in launches]
    tt = sum(t) or 1.0
    dram = [m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in launches]
    dm = sum(m.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * ti
             for m, ti in zip(launches, t)) / tt
    fp = sum(m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * ti
             for m, ti in zip(launches, t)) / tt
    rec = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            rec = json.load(fh)
    rec[wl] = {"kernel_regex": pat, "launches": n, "dram_bytes_per_launch": sum(dram) / max(n, 1),
               "dmma_pipe_pct": dm, "fp64_pipe_pct": fp, "ncu_ms_total": tt * 1e3, "source": src}
    with open(OUT, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(wl, rec[wl])


if __name__ == "__main__":
    main()
