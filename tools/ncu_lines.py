"""Aggregate ncu warp-stall samples by CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys


def main(path, top=25):
    cur_file = None
    out = []
    for r in csv.reader(open(path)):
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0].isdigit():
            try:
                out.append((int(float(r[4])), cur_file, r[0], r[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(o[0] for o in out) or 1
    print("total samples", tot)
    for s, f, ln, txt in sorted(out, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}%  {f}:{ln}  {txt}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
