"""One-off extractor: the paper's printed 12-node example matrices -> text
fixtures in this directory.  Run manually (``python
tests/golden/extract_paper_example.py /root/reference/PAPER.md``); the
outputs are committed, so nothing reads PAPER.md at test time.

Every value written is the paper's own print (arXiv 2211.13706 PAPER.md):

  A.txt      adjacency matrix A              P:L161-178 (§2.2 "An example")
  Z.txt      zeta matrix Z                   P:L180-196 (Eq. zm)
  M.txt      Moebius matrix M                P:L197-212 (Eq. zm)
  N.txt      niv matrix N, 'inf' = ∞         P:L294-323 (§2.4)
  U.txt, V.txt  factors of Z = UV            P:L423-473 (Eq. zuv)
  B.txt      block matrix B = P V P^-1       P:L478-494 (Eq. exb)
  Binv.txt   B^-1
  Vinv.txt   V^-1 = P^-1 B^-1 P
"""
import re
import sys
import os


def _cell(tok: str) -> str:
    t = tok.replace("\\phantom{-}", "").replace("\\phantom{1}", "").replace("\\zeroel", "0")
    t = t.replace("\\cdot", "0").replace("\\?", "").strip()
    if t == "":
        return "0"
    if t == "\\infty":
        return "inf"
    return t


def _matrix(body: str):
    rows = []
    for line in body.split("\\\\"):
        line = line.strip()
        if not line or line in ("\\phantom{1}",):
            continue
        cells = [_cell(c) for c in line.split("&")]
        if all(c == "0" for c in cells) and len(cells) == 1:
            continue
        rows.append(cells)
    return rows


def main(path):
    lines = open(path, encoding="utf-8").read().split("\n")
    out_dir = os.path.dirname(os.path.abspath(__file__))

    def grab(start, end, opener):
        """Matrix between 1-based lines [start, end] after ``opener``."""
        text = "\n".join(lines[start - 1:end])
        i = text.index(opener) + len(opener)
        j = text.index("\\end{psmallmatrix}", i)
        return _matrix(text[i:j]), text[j + len("\\end{psmallmatrix}"):]

    def write(name, rows, cite):
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(f"# {cite}\n")
            for r in rows:
                f.write(" ".join(r) + "\n")

    A, _ = grab(161, 178, "\\begin{psmallmatrix}")
    write("A.txt", A, "PAPER.md P:L161-178, adjacency matrix A of the 12-node example (§2.2)")
    Z, rest = grab(180, 212, "Z=\\begin{psmallmatrix}")
    write("Z.txt", Z, "PAPER.md P:L180-196, Eq. (zm) Z")
    M, _ = grab(197, 212, "M=\\begin{psmallmatrix}")
    write("M.txt", M, "PAPER.md P:L197-212, Eq. (zm) M")
    # N uses xsmallmatrix
    text = "\n".join(lines[293:311])
    i = text.index("\\begin{xsmallmatrix}{1em}") + len("\\begin{xsmallmatrix}{1em}")
    j = text.index("\\end{xsmallmatrix}")
    N = [r for r in _matrix(text[i:j]) if not any("phantom" in c for c in r)]
    write("N.txt", N, "PAPER.md P:L294-323, niv matrix N (columns Z1..Z4; 'inf' = infinity)")
    text = "\n".join(lines[422:473])
    parts = text.split("\\begin{psmallmatrix}")[1:]
    mats = [_matrix(p[:p.index("\\end{psmallmatrix}")]) for p in parts]
    write("U.txt", mats[1], "PAPER.md P:L441-456, Eq. (zuv) U")
    write("V.txt", mats[2], "PAPER.md P:L458-473, Eq. (zuv) V")
    B, _ = grab(478, 494, "B=\\begin{psmallmatrix}")
    write("B.txt", B, "PAPER.md P:L478-494, Eq. (exb) B = P V P^-1")
    Bi, _ = grab(506, 523, "B^{-1} =\\begin{psmallmatrix}")
    write("Binv.txt", Bi, "PAPER.md P:L506-523, B^-1")
    Vi, _ = grab(525, 542, "V^{-1} = P^{-1}B^{-1}P =\\begin{psmallmatrix}")
    write("Vinv.txt", Vi, "PAPER.md P:L525-542, V^-1 = P^-1 B^-1 P")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/PAPER.md")
