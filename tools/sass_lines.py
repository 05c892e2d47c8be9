"""Join an ncu SASS-page CSV (Instructions Executed, stall samples) with nvdisasm -g line info.
usage: sass_lines.py <ncu_sass.csv> <nvdisasm -g output> <mangled kernel name> [top]"""
import collections, csv, re, sys

csvp, disp, name = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = open(disp).read().split("\n")
i0 = [i for i, l in enumerate(txt) if l.startswith(".text." + name + ":")][0]
cur, lines = None, []
for l in txt[i0 + 1:]:
    if l.startswith("//----") or l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@{]", l):
        lines.append(cur)
rows = list(csv.reader(open(csvp)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ie, iw = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return int(x.replace(",", ""))
    except ValueError:
        return 0


data = []
for r in rows[hi + 1:]:
    if not r or not r[0].startswith("0x"):  # next section (another function) starts
        break
    data.append((num(r[ie]), num(r[iw])))
print("sass instructions", len(lines), "ncu rows", len(data))
agg = collections.defaultdict(lambda: [0, 0])
for (ins, st), ln in zip(data, lines):
    agg[ln][0] += ins
    agg[ln][1] += st
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print("instructions executed", ti, "stall samples", ts)
import os
root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2306_16778_b200", "csrc")
src = {}
for ln, (ins, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    s = ""
    if ln:
        if ln[0] not in src:
            p = os.path.join(root, ln[0])
            src[ln[0]] = open(p).read().split("\n") if os.path.exists(p) else []
        f = src[ln[0]]
        s = f[ln[1] - 1].strip()[:72] if ln[1] - 1 < len(f) else ""
    print(f"{ins / ti:6.3f} {st / max(ts, 1):6.3f} {ln} {s}")
