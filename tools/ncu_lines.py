"""Summarise an ncu --set full capture of engine_kernel by source line.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [iterations_per_launch] [top]

Prints, per CUDA source line, warp instructions executed per scheduler
iteration, average active threads, and the non-barrier stall samples (the
barrier samples are the warps idling while the critical-path warp works).
"""
import csv
import sys


def main():
    path = sys.argv[1]
    iters = float(sys.argv[2]) if len(sys.argv) > 2 else 250.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out, f, idx = [], None, None
    for r in csv.reader(open(path)):
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            idx = {h: i for i, h in enumerate(r)}
            continue
        if idx and r and r[0] not in ("", "Function Name"):
            try:
                ie = int(r[idx["Instructions Executed"]])
                ti = int(r[idx["Thread Instructions Executed"]])
            except (ValueError, KeyError):
                continue
            st = {h: int(r[i]) for h, i in idx.items()
                  if h.startswith("stall_") and "Not" not in h and r[i].isdigit()}
            nb = sum(v for k, v in st.items() if k != "stall_barrier")
            out.append((f, int(r[0]), r[1].strip()[:72], ie / iters, ti / max(ie, 1), nb))
    tot_ie = sum(o[3] for o in out)
    tot_nb = sum(o[5] for o in out)
    print(f"warp instructions / iteration: {tot_ie:.0f}; non-barrier stall samples: {tot_nb}")
    print(f"{'file':18s} line  instr/iter  threads  stalls(non-barrier)  source")
    for o in sorted(out, key=lambda x: (-x[5], -x[3]))[:top]:
        print(f"{o[0]:18s}{o[1]:5d} {o[3]:10.1f} {o[4]:8.1f} {o[5]:8d}   {o[2]}")


if __name__ == "__main__":
    main()
