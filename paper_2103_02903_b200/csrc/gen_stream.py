"""Generate stream_gen.cuh: fully unrolled flattened-table stream sums for the
built-in velocity sets (K7 fast path).

For every velocity set and gap class (0, 1, >= 2; the table offsets are identical
for every gap >= 2, asserted below up to gap 14) the generated function
  * loads the slots of all distinct table offsets of the class once per leaf,
  * per population loads each distinct operand once and evaluates
    sum_E then sum_A in table-entry order (lexicographic offsets, non-zero exact
    weights -- the order csrc/host_configs.cpp produces) with the weights taken
    from the runtime tables in shared memory,
so the arithmetic is identical to the generic table loop (and to the oracle).

Gap classes 0 and 1 take their weights as compile-time constants (exact dyadics,
rounded to nearest like csrc/host_configs.cpp; gen_w_* arrays let mrlbm_create
verify them against the runtime tables).  At gap 0 every weight and the scale
2^{d(l-J)} are exactly 1, so the multiplications by them are dropped (x * 1 == x
bit for bit).

The collision m = M f and f* = M^-1 m' is unrolled over the zero / +1 / -1 /
general pattern of the scheme's matrices (collide_patterns.json, written by
tools/collide_patterns.py): zero terms are skipped, +-1 terms become a plain
add / subtract (acc + 1*x == acc + x, acc + (-1)*x == acc - x exactly, and acc
starts at +0 so skipping +-0 products never changes it).  General entries are
read from the kernel-parameter copy of the matrices.  mrlbm_create checks the
runtime matrices against the pattern (gen_pat_*) before enabling this path.

Run: python paper_2103_02903_b200/csrc/gen_stream.py  (rewrites stream_gen.cuh)
"""
import itertools
import json
import os
from fractions import Fraction

C1 = Fraction(-1, 8)


def pred_w(d, delta):
    if d == 1:
        s = 1 if delta[0] == 0 else -1
        return {(-1,): -s * C1, (0,): Fraction(1), (1,): s * C1}
    s0 = 1 if delta[0] == 0 else -1
    s1 = 1 if delta[1] == 0 else -1
    w = {(0, 0): Fraction(1)}

    def add(k, v):
        w[k] = w.get(k, 0) + v
    add((1, 0), s0 * C1); add((-1, 0), -s0 * C1); add((0, 1), s1 * C1); add((0, -1), -s1 * C1)
    t = -s0 * s1 * C1 * C1
    add((1, 1), t); add((-1, 1), -t); add((1, -1), -t); add((-1, -1), t)
    return w


def table_offsets(d, g, eta, side):
    n = 2 ** g
    inb = lambda x: all(0 <= xi < n for xi in x)  # noqa: E731
    cur = {}
    for x in itertools.product(range(-1, n + 1), repeat=d):
        xe = tuple(xi + e for xi, e in zip(x, eta))
        if (inb(xe) and not inb(x)) if side == 0 else (inb(x) and not inb(xe)):
            cur[x] = Fraction(1)
    for _ in range(g):
        nxt = {}
        for c, w in cur.items():
            p = tuple(ci >> 1 for ci in c)
            dl = tuple(ci - 2 * pi for ci, pi in zip(c, p))
            for o, wo in pred_w(d, dl).items():
                k = tuple(pi + oi for pi, oi in zip(p, o))
                nxt[k] = nxt.get(k, 0) + w * wo
        cur = nxt
    return [k for k, v in sorted(cur.items()) if v != 0]


def table_weights_exact(d, g, eta, side):
    n = 2 ** g
    inb = lambda x: all(0 <= xi < n for xi in x)  # noqa: E731
    cur = {}
    for x in itertools.product(range(-1, n + 1), repeat=d):
        xe = tuple(xi + e for xi, e in zip(x, eta))
        if (inb(xe) and not inb(x)) if side == 0 else (inb(x) and not inb(xe)):
            cur[x] = Fraction(1)
    for _ in range(g):
        nxt = {}
        for c, w in cur.items():
            p = tuple(ci >> 1 for ci in c)
            dl = tuple(ci - 2 * pi for ci, pi in zip(c, p))
            for o, wo in pred_w(d, dl).items():
                k = tuple(pi + oi for pi, oi in zip(p, o))
                nxt[k] = nxt.get(k, 0) + w * wo
        cur = nxt
    return [float(v) for k, v in sorted(cur.items()) if v != 0]


def table_weights(d, g, etas):
    """All weights of one gap in table order (population, side, lexicographic offset)."""
    out = []
    for eta in etas:
        for side in (0, 1):
            out += table_weights_exact(d, g, eta, side)
    return out


D2Q4 = [(1, 0), (0, 1), (-1, 0), (0, -1)]
SETS = {
    # name: (d, q, eta list, equilibrium enum)
    "EQ1": (1, 2, [(1,), (-1,)]),
    "EQ2": (1, 9, [(0,), (1,), (-1,)] * 3),
    "EQ3": (2, 4, D2Q4),
    "EQ4": (2, 16, D2Q4 * 4),
    "EQ5": (2, 9, [(0, 0), (1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (-1, 1), (-1, -1), (1, -1)]),
}


def gen_class(name, d, q, etas, gclass, out):
    g = gclass
    tabs = {}
    for h, eta in enumerate(etas):
        for side in (0, 1):
            tabs[(h, side)] = table_offsets(d, g, eta, side)
            if gclass == 2:
                for gg in range(3, 15 if d == 1 else 11):
                    assert table_offsets(d, gg, eta, side) == tabs[(h, side)], (name, h, side, gg)
    offs = sorted({o for v in tabs.values() for o in v})
    oid = {o: i for i, o in enumerate(offs)}
    fn = f"gen_stream_{name}_g{gclass}"
    out.append(f"// {name}: gap class {gclass} ({len(offs)} distinct offsets)")
    out.append(f"__device__ __forceinline__ void {fn}(const double* __restrict__ Fin, long long cap, "
               f"int x, int y, int nx, int ny, int per0, int per1, "
               f"long long s, const double* sW, double scale, double (&f)[{q}])")
    out.append("{")
    out.append("    (void)y; (void)ny; (void)per1; (void)nx; (void)per0;")
    for o, i in oid.items():
        ox = o[0]
        oy = o[1] if d == 2 else 0
        xs = f"x + ({ox})" if ox else "x"
        # 32-bit linear indices (a level holds < 2^31 cells): half the registers of 64-bit ones
        if d == 1:
            out.append(f"    const int sl{i} = gen_wrap({xs}, nx, per0);")
        else:
            ys = f"y + ({oy})" if oy else "y"
            out.append(f"    const int sl{i} = gen_vix(gen_wrap({xs}, nx, per0), gen_wrap({ys}, ny, per1), ny);")
    widx = 0
    wts = table_weights(d, g, etas) if gclass < 2 else None
    for h in range(q):
        used = sorted({oid[o] for side in (0, 1) for o in tabs[(h, side)]})
        out.append("    {")
        out.append(f"        const double* Fh = Fin + {h}LL * cap;")
        out.append("        const double fs = Fh[s];")
        for u in used:
            out.append(f"        const double v{u} = Fh[sl{u}];")
        sums = []
        for side in (0, 1):
            nm = "sE" if side == 0 else "sA"
            out.append(f"        double {nm} = 0.0;")
            for o in tabs[(h, side)]:
                if gclass == 0:
                    assert wts[widx] == 1.0
                    out.append(f"        {nm} = __dadd_rn({nm}, v{oid[o]});")
                elif gclass == 1:
                    out.append(f"        {nm} = __dadd_rn({nm}, __dmul_rn({wts[widx].hex()}, v{oid[o]}));")
                else:
                    out.append(f"        {nm} = __dadd_rn({nm}, __dmul_rn(sW[{widx}], v{oid[o]}));")
                widx += 1
            sums.append(nm)
        if gclass == 0:
            out.append(f"        f[{h}] = __dadd_rn(fs, __dsub_rn(sE, sA));")
        else:
            out.append(f"        f[{h}] = __dadd_rn(fs, __dmul_rn(scale, __dsub_rn(sE, sA)));")
        out.append("    }")
    out.append("}")
    out.append("")
    if gclass < 2:
        out.append(f"static const double gen_w_{name}_g{gclass}[{len(wts)}] = {{{', '.join(w.hex() for w in wts)}}};")
        out.append("")
    return widx


def rim_cells_g1(d, eta, side):
    """E (side 0) / A (side 1) finest cells of a gap-1 leaf, lexicographic, as
    offsets (dx, dy) in the 4^d box [2x-1, 2x+3) x [2y-1, 2y+3)."""
    out = []
    rng = range(0, 4)
    inb = lambda c: all(1 <= ci <= 2 for ci in c)  # noqa: E731
    for c in itertools.product(rng, repeat=d):
        ce = tuple(ci + e for ci, e in zip(c, eta))
        if (inb(ce) and not inb(c)) if side == 0 else (inb(c) and not inb(ce)):
            out.append(c)
    return out


def gen_fb1h(name, d, q, etas, out):
    """Gap-1 fallback leaves, one population (one warp per population in k_fb1,
    selected by a warp-uniform switch on h): table sums + details of the rim cells
    that are finest leaves (Decision D.13b), per side selected by the masks; box =
    5^d level-l linear indices, rim = 4^d finest linear indices of leaves (-1: not a
    leaf); dmask pairs are left to the caller."""
    tabs = {(h, side): table_offsets(d, 1, eta, side) for h, eta in enumerate(etas) for side in (0, 1)}
    bidx = (lambda o: o[0] + 2) if d == 1 else (lambda o: (o[0] + 2) * 5 + (o[1] + 2))
    out.append(f"__device__ __forceinline__ void gen_fb1h_{name}(int h, const double* __restrict__ Fin, long long cap, "
               f"const double* __restrict__ Fj, long long capj, const int* box, const int* rim, int bstride, "
               f"unsigned mask, unsigned dmask, const double* sW, double& sE, double& sA)")
    out.append("{")
    out.append("    switch (h)")
    out.append("    {")
    widx = 0
    for h, eta in enumerate(etas):
        needed_box = set()
        for side in (0, 1):
            for o in tabs[(h, side)]:
                needed_box.add(bidx(o))
        out.append(f"    case {h}:")
        out.append("    {")
        out.append(f"        const double* Fh = Fin + {h}LL * cap;")
        out.append(f"        const double* Fjh = Fj + {h}LL * capj;")
        out.append("        (void)Fjh; (void)Fh;")
        for b in sorted(needed_box):
            out.append(f"        const double v{b} = Fh[box[{b} * bstride]];")
        for side in (0, 1):
            nm = "sE" if side == 0 else "sA"
            pair = 2 * h + side
            out.append(f"        if (!((dmask >> {pair}) & 1u))")
            out.append("        {")
            out.append("            double acc = 0.0;")
            for o in tabs[(h, side)]:
                out.append(f"            acc = __dadd_rn(acc, __dmul_rn(sW[{widx}], v{bidx(o)}));")
                widx += 1
            rims = rim_cells_g1(d, eta, side)
            if rims:
                out.append(f"            if ((mask >> {pair}) & 1u)")
                out.append("            {")
                extra = set()
                for c in rims:
                    p = tuple((ci + 1) // 2 - 1 for ci in c)
                    for st in itertools.product((-1, 0, 1), repeat=d):
                        extra.add(bidx(tuple(pi + si for pi, si in zip(p, st))))
                for b in sorted(extra - needed_box):
                    out.append(f"                const double v{b} = Fh[box[{b} * bstride]];")
                for c in rims:
                    r = c[0] if d == 1 else c[0] * 4 + c[1]
                    p = tuple((ci + 1) // 2 - 1 for ci in c)
                    par = tuple((ci + 1) & 1 for ci in c)
                    out.append("                {")
                    out.append(f"                    const int sj = rim[{r} * bstride];")
                    out.append("                    if (sj >= 0)")
                    out.append("                    {")
                    sv = [f"v{bidx(tuple(pi + si for pi, si in zip(p, st)))}" for st in itertools.product((-1, 0, 1), repeat=d)]
                    out.append(f"                        const double sv[{len(sv)}] = {{{', '.join(sv)}}};")
                    dy = par[1] if d == 2 else 0
                    out.append(f"                        acc = __dadd_rn(acc, __dsub_rn(Fjh[sj], mr_predict<{d}>(sv, {par[0]}, {dy})));")
                    out.append("                    }")
                    out.append("                }")
                out.append("            }")
            out.append(f"            {nm} = acc;")
            out.append("        }")
        out.append("        break;")
        out.append("    }")
    out.append("    default:")
    out.append("        break;")
    out.append("    }")
    out.append("}")
    out.append("")


def gen_matvec(fn, name, q, bs, pat, arr, src, dst, out):
    """dst[i] = sum_c A[i][b0 + c] * src[b0 + c] over the pattern, DenseMatrix::multiply order."""
    out.append(f"template <class CC>")
    out.append(f"__device__ __forceinline__ void {fn}_{name}(const CC& cc, const double (&{src})[{q}], double (&{dst})[{q}])")
    out.append("{")
    for i in range(q):
        b0 = (i // bs) * bs
        terms = []
        for c, ch in enumerate(pat[i]):
            j = b0 + c
            if ch == "0":
                continue
            if ch == "+":
                terms.append(("add", f"{src}[{j}]"))
            elif ch == "-":
                terms.append(("sub", f"{src}[{j}]"))
            else:
                terms.append(("add", f"__dmul_rn(cc.{arr}[{i * bs + c}], {src}[{j}])"))
        if not terms:
            out.append(f"    {dst}[{i}] = 0.0;")
            continue
        expr = "0.0"
        for op, t in terms:
            expr = f"__d{op}_rn({expr}, {t})"
        out.append(f"    {dst}[{i}] = {expr};")
    out.append("}")
    out.append("")


def gen_matrow(fn, name, q, bs, pat, arr, out):
    """Row i of the same product (warp-uniform switch), for the row-per-warp collision of k_fb1."""
    out.append("template <class CC>")
    out.append(f"__device__ __forceinline__ double {fn}_row_{name}(const CC& cc, int i, const double (&x)[{q}])")
    out.append("{")
    out.append("    switch (i)")
    out.append("    {")
    for i in range(q):
        b0 = (i // bs) * bs
        expr = None
        for c, ch in enumerate(pat[i]):
            j = b0 + c
            if ch == "0":
                continue
            t = f"x[{j}]" if ch in "+-" else f"__dmul_rn(cc.{arr}[{i * bs + c}], x[{j}])"
            op = "sub" if ch == "-" else "add"
            expr = f"__d{op}_rn({expr or '0.0'}, {t})"
        out.append(f"    case {i}:")
        out.append(f"        return {expr or '0.0'};")
    out.append("    default:")
    out.append("        return 0.0;")
    out.append("    }")
    out.append("}")
    out.append("")


def gen_collide(out):
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "collide_patterns.json")
    pats = json.load(open(path))
    for name in SETS:
        p = pats[name]
        q, bs = p["q"], p["bs"]
        gen_matvec("gen_mf", name, q, bs, p["M"], "M", "f", "m", out)
        gen_matvec("gen_minv", name, q, bs, p["Minv"], "Mi", "m", "f", out)
        gen_matrow("gen_mf", name, q, bs, p["M"], "M", out)
        gen_matrow("gen_minv", name, q, bs, p["Minv"], "Mi", out)
        out.append(f'static const char gen_pat_{name}_M[] = "{"".join(p["M"])}";')
        out.append(f'static const char gen_pat_{name}_Minv[] = "{"".join(p["Minv"])}";')
        out.append("")


def gen_fb1t(name, d, q, etas, out, rs=False):
    """Gap-1 fallback leaves, one thread per leaf (k_fb1t): every population's
    table sums + details of the rim cells that are finest leaves (Decision D.13b),
    the same operands and order as gen_fb1h.  For leaves without domain-leaving
    pairs (dmask == 0): box values are loaded at clamped / wrapped coordinates (the
    pairs that use them are inside the domain), rim cells are tested for finest
    leaves on the fly."""
    tabs = {(h, side): table_offsets(d, 1, eta, side) for h, eta in enumerate(etas) for side in (0, 1)}
    box = [o for o in itertools.product(range(-2, 3), repeat=d)]
    bidx = (lambda o: o[0] + 2) if d == 1 else (lambda o: (o[0] + 2) * 5 + (o[1] + 2))
    if rs:
        # boundary-rim variant: pairs whose dependencies leave the domain take rs(h, side)
        # (the recursive rim sum with the boundary rule) instead of table + details
        out.append("template <class RS>")
        out.append(f"__device__ __forceinline__ void gen_fb1t_rs_{name}(const double* __restrict__ Fin, long long cap, "
                   f"const double* __restrict__ Fj, long long capj, unsigned ring, "
                   f"int x, int y, int nx, int ny, int nxj, int nyj, int per0, int per1, unsigned mask, unsigned dmask, "
                   f"const RS& rs, long long s, const double* sW, double scale, double (&f)[{q}])")
    else:
        out.append(f"__device__ __forceinline__ void gen_fb1t_{name}(const double* __restrict__ Fin, long long cap, "
                   f"const double* __restrict__ Fj, long long capj, unsigned ring, "
                   f"int x, int y, int nx, int ny, int nxj, int nyj, int per0, int per1, unsigned mask, "
                   f"long long s, const double* sW, double scale, double (&f)[{q}])")
    out.append("{")
    out.append("    (void)y; (void)ny; (void)nyj; (void)per1; (void)capj; (void)Fj; (void)ring; (void)nxj;")
    used_all = set()
    for h, eta in enumerate(etas):
        for side in (0, 1):
            for o in tabs[(h, side)]:
                used_all.add(bidx(o))
            for c in rim_cells_g1(d, eta, side):
                p = tuple((ci + 1) // 2 - 1 for ci in c)
                for st in itertools.product((-1, 0, 1), repeat=d):
                    used_all.add(bidx(tuple(pi + si for pi, si in zip(p, st))))
    for o in box:
        b = bidx(o)
        if b not in used_all:
            continue
        xs = f"x + ({o[0]})" if o[0] else "x"
        if d == 1:
            out.append(f"    const int b{b} = gen_clampw({xs}, nx, per0);")
        else:
            ys = f"y + ({o[1]})" if o[1] else "y"
            out.append(f"    const int b{b} = gen_vix(gen_clampw({xs}, nx, per0), gen_clampw({ys}, ny, per1), ny);")
    widx = 0
    for h, eta in enumerate(etas):
        out.append("    {")
        out.append(f"        const double* Fh = Fin + {h}LL * cap;")
        out.append(f"        const double* Fjh = Fj + {h}LL * capj;")
        out.append("        (void)Fjh;")
        out.append("        const double fs = Fh[s];")
        needed = sorted({bidx(o) for side in (0, 1) for o in tabs[(h, side)]})
        for b in needed:
            out.append(f"        const double v{b} = Fh[b{b}];")
        for side in (0, 1):
            nm = "sE" if side == 0 else "sA"
            pair = 2 * h + side
            out.append(f"        double {nm} = 0.0;")
            for o in tabs[(h, side)]:
                out.append(f"        {nm} = __dadd_rn({nm}, __dmul_rn(sW[{widx}], v{bidx(o)}));")
                widx += 1
            rims = rim_cells_g1(d, eta, side)
            if rims:
                out.append(f"        if ((mask >> {pair}) & 1u)")
                out.append("        {")
                extra = set()
                for c in rims:
                    p = tuple((ci + 1) // 2 - 1 for ci in c)
                    for st in itertools.product((-1, 0, 1), repeat=d):
                        extra.add(bidx(tuple(pi + si for pi, si in zip(p, st))))
                for b in sorted(extra - set(needed)):
                    out.append(f"            const double v{b} = Fh[b{b}];")
                for c in rims:
                    p = tuple((ci + 1) // 2 - 1 for ci in c)
                    par = tuple((ci + 1) & 1 for ci in c)
                    xs = f"2 * x + ({c[0] - 1})"
                    r = c[0] if d == 1 else c[0] * 4 + c[1]
                    # ring bit r: the finest cell is a leaf (computed once per leaf by the caller)
                    out.append(f"            if ((ring >> {r}) & 1u)")
                    out.append("            {")
                    if d == 1:
                        out.append(f"              const int jv = gen_wrap({xs}, nxj, per0);")
                    else:
                        ys = f"2 * y + ({c[1] - 1})"
                        out.append(f"              const int jv = gen_vix(gen_wrap({xs}, nxj, per0), gen_wrap({ys}, nyj, per1), nyj);")
                    out.append("              {")
                    sv = [f"v{bidx(tuple(pi + si for pi, si in zip(p, st)))}" for st in itertools.product((-1, 0, 1), repeat=d)]
                    out.append(f"                const double sv[{len(sv)}] = {{{', '.join(sv)}}};")
                    dy = par[1] if d == 2 else 0
                    out.append(f"                {nm} = __dadd_rn({nm}, __dsub_rn(Fjh[jv], mr_predict<{d}>(sv, {par[0]}, {dy})));")
                    out.append("              }")
                    out.append("            }")
                out.append("        }")
            if rs:
                out.append(f"        if ((dmask >> {pair}) & 1u)")
                out.append(f"            {nm} = rs({h}, {side});")
        out.append(f"        f[{h}] = __dadd_rn(fs, __dmul_rn(scale, __dsub_rn(sE, sA)));")
        out.append("    }")
    out.append("}")
    out.append("")


def main():
    out = ["// GENERATED by gen_stream.py -- do not edit.",
           "// Unrolled flattened-table stream sums for the built-in velocity sets (K7 fast path).",
           "#pragma once",
           "",
           "__device__ __forceinline__ int gen_wrap(int c, int n, int per)",
           "{",
           "    return per ? (c < 0 ? c + n : (c >= n ? c - n : c)) : c;",
           "}",
           "",
           "// value index in 2x2 sibling blocks (2D layout, mrlbm_step.cu vix)",
           "__device__ __forceinline__ int gen_vix(int x, int y, int ny)",
           "{",
           "    return (((x >> 1) * (ny >> 1) + (y >> 1)) << 2) + ((x & 1) << 1) + (y & 1);",
           "}",
           "",
           "// MR boundary rule (Decision D.8): wrap periodic axes, clamp the others",
           "__device__ __forceinline__ int gen_clampw(int c, int n, int per)",
           "{",
           "    return per ? (c < 0 ? c + n : (c >= n ? c - n : c)) : (c < 0 ? 0 : (c >= n ? n - 1 : c));",
           "}",
           ""]
    for name, (d, q, etas) in SETS.items():
        for gc in (0, 1, 2):
            gen_class(name, d, q, etas, gc, out)
    for name, (d, q, etas) in SETS.items():
        gen_fb1h(name, d, q, etas, out)
    for name, (d, q, etas) in SETS.items():
        gen_fb1t(name, d, q, etas, out)
        gen_fb1t(name, d, q, etas, out, rs=True)
    gen_collide(out)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "stream_gen.cuh")
    open(path, "w").write("\n".join(out) + "\n")
    print("wrote", path, len(out), "lines")


if __name__ == "__main__":
    main()
