"""Aggregate an ncu source-page SASS export by CUDA source line.

    nvdisasm -gi ef_trace.sm_100a.cubin > all.sass
    ncu -i rep --page source --csv --print-source sass > k.csv
    python tools/sass_lines.py all.sass <mangled kernel name> k.csv [top]

Prints instructions executed / stall samples per (file, line), innermost
inline location first, with the source text."""
import csv
import re
import sys
from collections import defaultdict


def line_map(sass_path, kernel):
    amap, cur, inside, fresh = {}, None, False, True
    for l in open(sass_path):
        if l.startswith(kernel + ":"):
            inside = True
            continue
        if inside and l.startswith("//----"):
            break
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
        if m:
            if fresh:   # innermost location comes first
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                fresh = False
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m:
            amap[int(m.group(1), 16)] = cur
            fresh = True
    return amap


def main():
    sass, kernel, csv_path = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    amap = line_map(sass, kernel)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    inst, stall = defaultdict(int), defaultdict(int)
    tot_i = tot_s = 0
    for r in rows[2:]:
        try:
            a = int(r[ia], 16) - base
        except ValueError:
            continue
        loc = amap.get(a, ("?", 0))
        n = int(float(r[ie] or 0))
        s = int(float(r[iss] or 0))
        inst[loc] += n
        stall[loc] += s
        tot_i += n
        tot_s += s
    src = {}
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    for loc, n in sorted(inst.items(), key=lambda x: -x[1])[:top]:
        f, ln = loc
        if f not in src:
            try:
                src[f] = open("paper_1803_00430_b200/csrc/" + f).read().splitlines()
            except OSError:
                src[f] = []
        text = src[f][ln - 1].strip() if 0 < ln <= len(src[f]) else ""
        print(f"{n:8d} {100*n/tot_i:5.1f}%  stall {100*stall[loc]/max(tot_s,1):5.1f}%  {f}:{ln:<5d} {text[:90]}")


if __name__ == "__main__":
    main()
