"""Decode PAPER.md Fig. 1 (the TikZ block structures for a 1-D line of
n = 4, 8, 16 facets with n_min = 1) into text fixtures fig1_n{4,8,16}.txt.

Run once in the build container (the paper is not on the GPU box):
    python tests/golden/extract_fig1.py /root/reference/PAPER.md
Each `\\filldraw(x0,y0) [Rfill|Gfill] rectangle (x1,y1)` is a block; the picture is
3.2 units wide, so one facet is 3.2/n units; row = (3.2 - y_top)/cell, col = x0/cell.
Rfill (blue) = dense, Gfill (gray) = low-rank (caption PAPER.md:587).
"""
import re
import sys
from pathlib import Path

RECT = re.compile(r"\\filldraw\(([\d.]+),([\d.]+)\)\s*\[(Rfill|Gfill)\]\s*rectangle\s*\(([\d.]+),([\d.]+)\)")


def main(paper: str):
    lines = Path(paper).read_text().splitlines()
    fig = lines[370:589]
    pics, cur = [], []
    for ln in fig:
        m = RECT.search(ln)
        if m:
            cur.append(m.groups())
        if "end{tikzpicture}" in ln and cur:
            pics.append(cur)
            cur = []
    out = Path(__file__).parent
    for blocks in pics:
        n = {16: 4, 46: 8, 112: 16}[len(blocks)]
        cell = 3.2 / n
        rows = []
        for x0, y0, kind, x1, y1 in blocks:
            x0, y0, x1, y1 = map(float, (x0, y0, x1, y1))
            r0 = round((3.2 - y1) / cell)
            r1 = round((3.2 - y0) / cell)
            c0 = round(x0 / cell)
            c1 = round(x1 / cell)
            rows.append((r0, r1, c0, c1, 1 if kind == "Gfill" else 0))
        rows.sort()
        with open(out / f"fig1_n{n}.txt", "w") as f:
            f.write(f"# PAPER.md Fig. 1 (lines 371-589), n={n}, n_min=1; decoded by extract_fig1.py\n")
            f.write("# row_begin row_end col_begin col_end admissible(1=low-rank gray, 0=dense blue)\n")
            for r in rows:
                f.write(" ".join(map(str, r)) + "\n")
        print(n, len(rows), sum(r[4] for r in rows))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/PAPER.md")
