"""Hot instruction footprint of a kernel from an ncu source export.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_hot_lines.py src.csv [iterations_per_launch]

Groups the executed SASS by 128-byte instruction-cache line and by CUDA
source region, and reports the lines executed at least once per scheduler
iteration (the per-iteration instruction footprint the L1.5 cache must hold),
with how many of those are executed by a single thread (serial sections).
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    iters = float(sys.argv[2]) if len(sys.argv) > 2 else 250.0
    idx, f, src = None, None, None
    ins = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            idx = {h: i for i, h in enumerate(r)}
            continue
        if not idx or not r:
            continue
        if r[0] not in ("",):
            try:
                src = (f, int(r[0]))
            except ValueError:
                pass
            continue
        try:
            addr = int(r[2], 16)
            ex = int(r[idx["Instructions Executed"]])
            th = float(r[idx["Avg. Threads Executed"]] or 0)
        except (ValueError, KeyError, IndexError):
            continue
        if addr not in ins or ex > ins[addr][0]:
            ins[addr] = (ex, th, src, r[3])
    lines = collections.defaultdict(list)
    for a, v in ins.items():
        lines[a >> 7].append(v)
    hot = {k: v for k, v in lines.items() if max(x[0] for x in v) >= iters}
    print(f"instructions: {len(ins)}; executed: {sum(1 for v in ins.values() if v[0])}; "
          f"128-B lines executed >= once per iteration: {len(hot)} ({len(hot) * 128 / 1024:.1f} KB)")
    serial = {k: v for k, v in hot.items() if max(x[1] for x in v if x[0]) <= 1.5}
    print(f"  of which single-thread lines: {len(serial)}")
    by = collections.Counter()
    for k, v in hot.items():
        srcs = collections.Counter(x[2] for x in v if x[0] >= iters)
        s = srcs.most_common(1)[0][0] if srcs else None
        by[(s[0], s[1] // 10 * 10) if s else None] += 1
    print("hot lines by source region (file, line//10*10):")
    for k, n in by.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 40):
        print(f"  {str(k):40s} {n}")


if __name__ == "__main__":
    main()
