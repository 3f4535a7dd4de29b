"""Aggregate an ncu source page (--print-source cuda,sass CSV) per CUDA line.

    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top] [--by-ins]
(--by-ins: lines ordered by executed warp instructions instead of stall samples)"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    args = [a for a in sys.argv[2:] if not a.startswith("--")]
    by_ins = "--by-ins" in sys.argv
    top = int(args[0]) if args else 40
    out = []
    fname = None
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[0] == "" or r[0] == "Function Name":
            continue
        try:
            samples = float(r[4] or 0)
            ins = float(r[7] or 0)
            thr = float(r[8] or 0)
        except ValueError:
            continue
        out.append((samples, ins, thr, f"{fname}:{r[0]}", r[1][:90]))
    tot = sum(o[0] for o in out) or 1
    tins = sum(o[1] for o in out) or 1
    out.sort(key=(lambda o: o[1]) if by_ins else (lambda o: o[0]), reverse=True)
    print(f"total stall samples {tot:.0f}, warp instructions {tins:.3g}")
    for s, i, t, loc, src in out[:top]:
        act = t / i if i else 0
        print(f"{100 * s / tot:5.1f}%  ins {100 * i / tins:5.1f}%  act {act:4.1f}  {loc:22s} {src}")


if __name__ == "__main__":
    main()
