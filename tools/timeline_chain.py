"""Critical-chain breakdown from a PFX_PROF_TIMELINE dump (pfx_api.cu prof_read).

Usage: python tools/timeline_chain.py <timeline.txt> [anchor_kernel]
Takes the last '# timeline' block; the stream that launches the anchor kernel (default
zgetrf_diag, the band LU's diagonal factorisation) is the critical chain.  Prints, per kernel
name on that stream, the mean duration, and the mean gap between consecutive chain launches,
plus the mean step period (anchor start to anchor start)."""
import sys
from collections import defaultdict


def main(path, anchor="zgetrf_diag"):
    blocks, cur = [], None
    for line in open(path):
        if line.startswith("# timeline"):
            cur = []
            blocks.append(cur)
        elif cur is not None and line.strip():
            name, st, a, b = line.split()
            cur.append((name, st, float(a), float(b)))
    recs = blocks[-1]
    main_st = next(st for n, st, _, _ in recs if n.split("@")[0] == anchor)
    chain = sorted([r for r in recs if r[1] == main_st], key=lambda r: r[2])
    dur, gaps_after = defaultdict(list), defaultdict(list)
    for i, (n, _, a, b) in enumerate(chain):
        dur[n].append(b - a)
        if i + 1 < len(chain):
            gaps_after[n].append(chain[i + 1][2] - b)
    starts = [a for n, _, a, _ in chain if n.split("@")[0] == anchor]
    period = (starts[-1] - starts[0]) / max(1, len(starts) - 1) if len(starts) > 1 else float("nan")
    span = chain[-1][3] - chain[0][2]
    print(f"records {len(recs)}  chain launches {len(chain)}  span {span / 1e3:.2f} ms  "
          f"anchor steps {len(starts)}  period {period:.2f} us")
    print(f"{'kernel':28s} {'n':>6s} {'mean us':>9s} {'sum ms':>9s} {'gap after us':>13s}")
    for n in sorted(dur, key=lambda k: -sum(dur[k])):
        g = gaps_after[n]
        print(f"{n:28s} {len(dur[n]):6d} {sum(dur[n]) / len(dur[n]):9.2f} {sum(dur[n]) / 1e3:9.2f} "
              f"{(sum(g) / len(g) if g else 0):13.2f}")
    other = defaultdict(lambda: [0, 0.0])
    for n, st, a, b in recs:
        if st != main_st:
            other[(n, st)][0] += 1
            other[(n, st)][1] += b - a
    print("off-chain streams:")
    for (n, st), (c, t) in sorted(other.items(), key=lambda x: -x[1][1])[:12]:
        print(f"  {n:26s} {st:>16s} {c:6d} {t / c:9.2f} us  {t / 1e3:9.2f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
