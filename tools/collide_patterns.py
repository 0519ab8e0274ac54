"""Write paper_2103_02903_b200/csrc/collide_patterns.json: the zero / +1 / -1 / general
pattern of M and M^-1 (block-diagonal compact layout, row i, column within the block)
of the five BASELINE schemes, taken from the built library's own config builders.

gen_stream.py turns the patterns into unrolled collision code; mrlbm_create checks
at run time that a scheme's matrices fit the pattern (else the generic path runs).
Run after building: python tools/collide_patterns.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_02903_b200 import build_config  # noqa: E402


def pattern(vals, q, bs):
    out = []
    for i in range(q):
        b0 = (i // bs) * bs
        row = ""
        for c in range(bs):
            v = vals[i * q + b0 + c]
            row += "0" if v == 0.0 else ("+" if v == 1.0 else ("-" if v == -1.0 else "G"))
        out.append(row)
    return out


def main():
    pats = {}
    for cid in range(1, 6):
        sc, _ = build_config(cid, 0)
        q, bs = sc.q, sc.q // sc.nblocks
        pats[f"EQ{sc.equilibrium}"] = {"q": q, "bs": bs, "M": pattern(sc.M, q, bs), "Minv": pattern(sc.Minv, q, bs)}
    path = os.path.join(ROOT, "paper_2103_02903_b200", "csrc", "collide_patterns.json")
    with open(path, "w") as fh:
        json.dump(pats, fh, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
