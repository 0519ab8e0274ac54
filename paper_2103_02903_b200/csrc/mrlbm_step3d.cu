// mrlbm_step3d.cu — the 3D adaptive MR-LBM time step (the D3Q6 path of
// PAPER.md:1462-1518), hand-written CUDA for sm_100a behind the same
// C-ABI (mrlbm_create with scheme.d == 3 builds this engine).
//
// Same algorithm and the same floating-point operation order as the 1D/2D step in
// mrlbm_step.cu (Algorithm 1 body; decisions D.1-D.27 of DESIGN.md),
// with the reference's 3D prediction operator (prediction.hpp:160-172: three axis terms,
// three plane terms subtracted, one triple term) and 2^3 sibling groups.
//
// Layout (per level l, box nx x ny x nz, lexicographic linear index, axis 0 slow):
//   kind[v][l]  uint8 dense: bit 0 complete leaf, bit 1 internal node of tree version v
//   F[b][l]     fp64 dense, one contiguous array per population: F[h * n + lin]
//   keep, rn    uint8 dense per-step flags (T_eps groups at the parent, refined cells)
// After the transfer and the projection of the new tree, F of the current buffer holds
// the zero-detail reconstruction f^^ on every cell the stream can
// touch: cells of the complete tree keep their value, the others are predicted top-down
// from level l-1 (the oracle's rec(), same operands and order).  The reconstruction is
// restricted to the cells marked needed (a top-down need mask seeded by the table
// stencils and the finest rims of the leaves).
//
// Velocity sets: |eta_i| <= 1 with at most one non-zero component per velocity (D3Q6 and
// its vectorial / rest-velocity variants); mrlbm_create returns status 2 otherwise.

#include "mrlbm_internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace mrlbm_b200 {

namespace {

constexpr int kL3 = MRLBM_MAX_LEVELS;
constexpr int kQ3 = MRLBM_MAX_Q;
constexpr uint8_t K3_LEAF = 1, K3_INT = 2;
constexpr int kTieCap3 = 1 << 16;
constexpr int kWarpGap3 = 2;  // levels with gap >= 2 (rims of >= 16 finest cells): one warp per leaf
constexpr int kBlockGap3 = 5; // levels with gap >= 5 (rims of >= 1024 cells): one block of 2 q warps per leaf
                              // (measured at J = 8: stream + collide 2233 us without, 2280 / 1990 / 1857 us from gap 3 / 4 / 5)

struct Geo3 {
    int J0, J1, nlev, q;
    int nx[kL3], ny[kL3], nz[kL3];
    long long n[kL3];
    int per[3];
};

struct Lv3 {
    uint8_t* kind[kL3];
};
struct Fl3 {
    double* f[kL3];
};
struct Bt3 {
    uint8_t* b[kL3];
};

// scheme constants on the device
struct Sch3 {
    int eta[kQ3][3];
    int opp[kQ3];
    double M[kQ3 * kQ3], Minv[kQ3 * kQ3], s[kQ3];
    double eqp[8];
    int equilibrium;
    int bc_kind[6];
    double bc_add[6][kQ3];
    double eps;
    int mu;
};

// flattened tables: per (gap, h, side) a range of (offset, weight) entries, the
// dependency bounding box and a range of parent offsets (Decision D.13)
struct Tab3 {
    const int2* tidx;   // [(g * q + h) * 2 + side] -> (start, count) into toff / tw
    const int* toff;    // 3 ints per entry
    const double* tw;
    const int* tdep;    // 6 ints per table: lo[3], hi[3]
    const int2* tpidx;  // -> (start, count) into tpar
    const int* tpar;    // 3 ints per parent offset
    const int* udep;    // 6 ints per gap: union of the dependency boxes (>= the 5^3 box at gap 1)
};

struct Aux3 {
    int* err;           // [0] unresolved stencil, [1] non-finite, [2] missing opposite velocity
    int* cnt;           // [2 * kL3] leaves, internal per level; [2 * kL3] fallback leaves
    mrlbm_tie_record* ties;
    int* tie_n;
    const int* step_no;
};

#define GS3(i, n) for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

__device__ __forceinline__ int coord3(int c, int n, int per)
{
    if (per)
    {
        c %= n;
        return c < 0 ? c + n : c;
    }
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

__device__ __forceinline__ void lin2xyz(const Geo3& g, int li, long long lin, int& x, int& y, int& z)
{
    // level boxes hold < 2^31 cells (checked at create): 32-bit divisions
    const unsigned ny = g.ny[li], nz = g.nz[li];
    const unsigned l = (unsigned)lin;
    const unsigned r = l / nz;
    z = (int)(l - r * nz);
    x = (int)(r / ny);
    y = (int)(r - (unsigned)x * ny);
}

__device__ __forceinline__ long long xyz2lin(const Geo3& g, int li, int x, int y, int z)
{
    return ((long long)x * g.ny[li] + y) * g.nz[li] + z;
}

// MR lookup rule (D.8): periodic wrap, else clamp to the nearest interior cell
__device__ __forceinline__ long long mr_lin3(const Geo3& g, int li, int x, int y, int z)
{
    return xyz2lin(g, li, coord3(x, g.nx[li], g.per[0]), coord3(y, g.ny[li], g.per[1]), coord3(z, g.nz[li], g.per[2]));
}

// reference predict<3> operation order (prediction.hpp:64-122, 160-172), gamma = 1.
// st[27]: stencil values, index (ox+1)*9 + (oy+1)*3 + (oz+1); (dx, dy, dz) child selector.
__device__ __forceinline__ double predict3(const double* st, int dx, int dy, int dz)
{
    const double c1 = -0.125;
    const double c2 = __dmul_rn(c1, c1);
    const double c3 = __dmul_rn(c2, c1);
#define ST(ox, oy, oz) st[((ox) + 1) * 9 + ((oy) + 1) * 3 + ((oz) + 1)]
    const double center = ST(0, 0, 0);
    const double s0 = dx == 0 ? 1.0 : -1.0, s1 = dy == 0 ? 1.0 : -1.0, s2 = dz == 0 ? 1.0 : -1.0;
    const double qx = __dadd_rn(0.0, __dmul_rn(c1, __dsub_rn(ST(1, 0, 0), ST(-1, 0, 0))));
    const double qy = __dadd_rn(0.0, __dmul_rn(c1, __dsub_rn(ST(0, 1, 0), ST(0, -1, 0))));
    const double qz = __dadd_rn(0.0, __dmul_rn(c1, __dsub_rn(ST(0, 0, 1), ST(0, 0, -1))));
    // q2(ax1, ax2): c c (at(pp) - at(mp) - at(pm) + at(mm)), mp = (-a on ax1, +b on ax2)
    const double ixy = __dadd_rn(__dsub_rn(__dsub_rn(ST(1, 1, 0), ST(-1, 1, 0)), ST(1, -1, 0)), ST(-1, -1, 0));
    const double ixz = __dadd_rn(__dsub_rn(__dsub_rn(ST(1, 0, 1), ST(-1, 0, 1)), ST(1, 0, -1)), ST(-1, 0, -1));
    const double iyz = __dadd_rn(__dsub_rn(__dsub_rn(ST(0, 1, 1), ST(0, -1, 1)), ST(0, 1, -1)), ST(0, -1, -1));
    const double qxy = __dadd_rn(0.0, __dmul_rn(c2, ixy));
    const double qxz = __dadd_rn(0.0, __dmul_rn(c2, ixz));
    const double qyz = __dadd_rn(0.0, __dmul_rn(c2, iyz));
    // q3: loop sx, sy, sz in {+, -} (sz fastest), sign + for an even number of minus
    double acc = 0.0;
    acc = __dadd_rn(acc, ST(1, 1, 1));
    acc = __dsub_rn(acc, ST(1, 1, -1));
    acc = __dsub_rn(acc, ST(1, -1, 1));
    acc = __dadd_rn(acc, ST(1, -1, -1));
    acc = __dsub_rn(acc, ST(-1, 1, 1));
    acc = __dadd_rn(acc, ST(-1, 1, -1));
    acc = __dadd_rn(acc, ST(-1, -1, 1));
    acc = __dsub_rn(acc, ST(-1, -1, -1));
    const double qxyz = __dadd_rn(0.0, __dmul_rn(c3, acc));
#undef ST
    double r = __dadd_rn(center, __dmul_rn(s0, qx));
    r = __dadd_rn(r, __dmul_rn(s1, qy));
    r = __dadd_rn(r, __dmul_rn(s2, qz));
    r = __dsub_rn(r, __dmul_rn(__dmul_rn(s0, s1), qxy));
    r = __dsub_rn(r, __dmul_rn(__dmul_rn(s0, s2), qxz));
    r = __dsub_rn(r, __dmul_rn(__dmul_rn(s1, s2), qyz));
    r = __dadd_rn(r, __dmul_rn(__dmul_rn(__dmul_rn(s0, s1), s2), qxyz));
    return r;
}

// 27-point stencil of population array fp (level li) around (px, py, pz), MR rule;
// ok = every stencil cell satisfies kind != 0 when kind is given
__device__ __forceinline__ bool load_stencil3(const Geo3& g, int li, const double* fp, const uint8_t* kind, int px,
                                              int py, int pz, double* st)
{
    bool ok = true;
    int xs[3], ys[3], zs[3];
#pragma unroll
    for (int o = 0; o < 3; ++o)
    {
        xs[o] = coord3(px + o - 1, g.nx[li], g.per[0]);
        ys[o] = coord3(py + o - 1, g.ny[li], g.per[1]);
        zs[o] = coord3(pz + o - 1, g.nz[li], g.per[2]);
    }
#pragma unroll
    for (int o = 0; o < 27; ++o)
    {
        const long long lin = xyz2lin(g, li, xs[o / 9], ys[(o / 3) % 3], zs[o % 3]);
        if (kind)
            ok = ok && kind[lin] != 0;
        st[o] = fp[lin];
    }
    return ok;
}

// the 27 linear indices of the stencil around (px, py, pz), MR rule, computed once per cell and
// reused for every population; ok = every stencil cell has kind != 0 when kind is given
__device__ __forceinline__ bool stencil_idx3(const Geo3& g, int li, const uint8_t* kind, int px, int py, int pz, int* lin)
{
    int xs[3], ys[3], zs[3];
#pragma unroll
    for (int o = 0; o < 3; ++o)
    {
        xs[o] = coord3(px + o - 1, g.nx[li], g.per[0]) * g.ny[li];
        ys[o] = coord3(py + o - 1, g.ny[li], g.per[1]);
        zs[o] = coord3(pz + o - 1, g.nz[li], g.per[2]);
    }
    bool ok = true;
#pragma unroll
    for (int o = 0; o < 27; ++o)
    {
        lin[o] = (xs[o / 9] + ys[(o / 3) % 3]) * g.nz[li] + zs[o % 3]; // < 2^31 cells per level box
        if (kind)
            ok = ok && kind[lin[o]] != 0;
    }
    return ok;
}

// ------------------------------------------------------------------ K1 / K6 projection
// internal node = mean of its 8 children in children order (prediction.hpp:51-60)
__global__ void __launch_bounds__(256) k3_project(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 t,
                                                  const __grid_constant__ Fl3 F, int li)
{
    const long long n = g.n[li], n1 = g.n[li + 1];
    const int ny1 = g.ny[li + 1], nz1 = g.nz[li + 1];
    GS3(i, n)
    {
        if (!(t.kind[li][i] & K3_INT))
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        const long long c0 = ((long long)(2 * x) * ny1 + 2 * y) * nz1 + 2 * z;
        for (int h = 0; h < g.q; ++h)
        {
            const double* src = F.f[li + 1] + (long long)h * n1;
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                s = __dadd_rn(s, src[c0 + ((long long)(c >> 2) * ny1 + ((c >> 1) & 1)) * nz1 + (c & 1)]);
            F.f[li][(long long)h * n + i] = __ddiv_rn(s, 8.0);
        }
    }
}

__device__ __forceinline__ void tie_check3(const Aux3& aux, int l, int px, int py, int pz, int which, double metric,
                                           double thr)
{
    if (thr > 0.0 && fabs(__dsub_rn(metric, thr)) <= __dmul_rn(1e-12, thr))
    {
        const int k = atomicAdd(aux.tie_n, 1);
        if (k < kTieCap3)
        {
            mrlbm_tie_record r;
            r.step = *aux.step_no + 1;
            r.level = l;
            r.cell[0] = px;
            r.cell[1] = py;
            r.cell[2] = pz;
            r.which = which;
            r.metric = metric;
            r.threshold = thr;
            aux.ties[k] = r;
        }
    }
}

// ------------------------------------------------------------------ K2 details
// d = f(child) - predict(parent stencil); group metric = max |d| over the 8 siblings and
// all populations; keep iff metric >= eps_l (Eq. 10), H(b) iff metric >= 2^(mu+d) eps_l
__global__ void __launch_bounds__(128) k3_details(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 t,
                                                  const __grid_constant__ Fl3 F, const __grid_constant__ Bt3 keep,
                                                  const __grid_constant__ Bt3 rn, const Sch3* sc, int li,
                                                  const __grid_constant__ Aux3 aux)
{
    const long long n = g.n[li], n1 = g.n[li + 1];
    const int ny1 = g.ny[li + 1], nz1 = g.nz[li + 1];
    const int l = g.J0 + li + 1;
    const double eps_l = ldexp(sc->eps, 3 * (l - g.J1));
    const double eps_b = ldexp(eps_l, sc->mu + 3);
    GS3(i, n)
    {
        if (!(t.kind[li][i] & K3_INT))
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        const long long c0 = ((long long)(2 * x) * ny1 + 2 * y) * nz1 + 2 * z;
        double metric = 0.0;
        int lin[27];
        const bool ok = stencil_idx3(g, li, t.kind[li], x, y, z, lin);
        for (int h = 0; h < g.q; ++h)
        {
            double st[27];
            const double* fp = F.f[li] + (long long)h * n;
#pragma unroll
            for (int o = 0; o < 27; ++o)
                st[o] = fp[lin[o]];
            const double* src = F.f[li + 1] + (long long)h * n1;
#pragma unroll
            for (int c = 0; c < 8; ++c)
            {
                const double cv = src[c0 + ((long long)(c >> 2) * ny1 + ((c >> 1) & 1)) * nz1 + (c & 1)];
                const double d = __dsub_rn(cv, predict3(st, c >> 2, (c >> 1) & 1, c & 1));
                const double ad = fabs(d);
                if (ad > metric)
                    metric = ad;
            }
        }
        if (!ok)
            atomicAdd(&aux.err[0], 1);
        if (metric >= eps_l)
            keep.b[li][i] = 1;
        const bool blow = l < g.J1;
        if (blow && metric >= eps_b)
        {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                rn.b[li + 1][c0 + ((long long)(c >> 2) * ny1 + ((c >> 1) & 1)) * nz1 + (c & 1)] = 1;
        }
        tie_check3(aux, l, x, y, z, 0, metric, eps_l);
        if (blow)
            tie_check3(aux, l, x, y, z, 1, metric, eps_b);
    }
}

// ------------------------------------------------------------------ K3 flags
// T closure (D.4): the parent of a kept cell is kept
__global__ void k3_closure(const __grid_constant__ Geo3 g, const __grid_constant__ Bt3 keep, int li)
{
    GS3(i, g.n[li])
    {
        if (!keep.b[li][i])
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        keep.b[li - 1][xyz2lin(g, li - 1, x >> 1, y >> 1, z >> 1)] = 1;
    }
}

// rn |= keep (R(T_eps)); H(a): for every cell c of R(T) at level li+1 (children of kept
// cells) and every velocity, the parent of c - eta is refined (clipped / wrapped), D.6
__global__ void k3_enlarge(const __grid_constant__ Geo3 g, const __grid_constant__ Bt3 keep,
                           const __grid_constant__ Bt3 rn, const Sch3* sc, int li)
{
    const int l1 = li + 1;
    GS3(i, g.n[li])
    {
        if (!keep.b[li][i])
            continue;
        rn.b[li][i] = 1;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        for (int c = 0; c < 8; ++c)
        {
            const int cx = 2 * x + (c >> 2), cy = 2 * y + ((c >> 1) & 1), cz = 2 * z + (c & 1);
            for (int h = 0; h < g.q; ++h)
            {
                const int ex = sc->eta[h][0], ey = sc->eta[h][1], ez = sc->eta[h][2];
                if (ex == 0 && ey == 0 && ez == 0)
                    continue;
                int sx = cx - ex, sy = cy - ey, sz = cz - ez;
                if (g.per[0])
                    sx = coord3(sx, g.nx[l1], 1);
                else if (sx < 0 || sx >= g.nx[l1])
                    continue;
                if (g.per[1])
                    sy = coord3(sy, g.ny[l1], 1);
                else if (sy < 0 || sy >= g.ny[l1])
                    continue;
                if (g.per[2])
                    sz = coord3(sz, g.nz[l1], 1);
                else if (sz < 0 || sz >= g.nz[l1])
                    continue;
                rn.b[li][xyz2lin(g, li, sx >> 1, sy >> 1, sz >> 1)] = 1;
            }
        }
    }
}

// grading G (D.7), one level of the fine -> coarse sweep: the parents of the 3^3 box
// (clipped / wrapped) of every refined cell of level li are refined
__global__ void k3_grade(const __grid_constant__ Geo3 g, const __grid_constant__ Bt3 rn, int li)
{
    GS3(i, g.n[li])
    {
        if (!rn.b[li][i])
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        for (int o = 0; o < 27; ++o)
        {
            int sx = x + o / 9 - 1, sy = y + (o / 3) % 3 - 1, sz = z + o % 3 - 1;
            if (g.per[0])
                sx = coord3(sx, g.nx[li], 1);
            else if (sx < 0 || sx >= g.nx[li])
                continue;
            if (g.per[1])
                sy = coord3(sy, g.ny[li], 1);
            else if (sy < 0 || sy >= g.ny[li])
                continue;
            if (g.per[2])
                sz = coord3(sz, g.nz[li], 1);
            else if (sz < 0 || sz >= g.nz[li])
                continue;
            rn.b[li - 1][xyz2lin(g, li - 1, sx >> 1, sy >> 1, sz >> 1)] = 1;
        }
    }
}

// ------------------------------------------------------------------ K4 kinds of the new tree
// R(J0) = the level box, R(l) = children of the refined cells; internal = refined
__global__ void k3_kinds(const __grid_constant__ Geo3 g, const __grid_constant__ Bt3 rn, const __grid_constant__ Lv3 tn,
                         int li, const __grid_constant__ Aux3 aux)
{
    __shared__ int sl, si;
    if (threadIdx.x == 0)
        sl = si = 0;
    __syncthreads();
    int nl = 0, ni = 0;
    GS3(i, g.n[li])
    {
        bool inR = li == 0;
        if (!inR)
        {
            int x, y, z;
            lin2xyz(g, li, i, x, y, z);
            inR = rn.b[li - 1][xyz2lin(g, li - 1, x >> 1, y >> 1, z >> 1)] != 0;
        }
        uint8_t k = 0;
        if (inR)
        {
            const bool internal = li < g.nlev - 1 && rn.b[li][i] != 0;
            k = internal ? K3_INT : K3_LEAF;
            nl += !internal;
            ni += internal;
        }
        tn.kind[li][i] = k;
    }
    atomicAdd(&sl, nl);
    atomicAdd(&si, ni);
    __syncthreads();
    if (threadIdx.x == 0)
    {
        if (sl)
            atomicAdd(&aux.cnt[2 * li], sl);
        if (si)
            atomicAdd(&aux.cnt[2 * li + 1], si);
    }
}

// ------------------------------------------------------------------ K5 transfer
// cells new to the complete tree: prediction from the new level li - 1
__global__ void __launch_bounds__(128) k3_transfer(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 to,
                                                   const __grid_constant__ Lv3 tn, const __grid_constant__ Fl3 F, int li,
                                                   const __grid_constant__ Aux3 aux)
{
    const long long n = g.n[li], np = g.n[li - 1];
    GS3(i, n)
    {
        if (!tn.kind[li][i] || to.kind[li][i])
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        int lin[27];
        const bool ok = stencil_idx3(g, li - 1, tn.kind[li - 1], x >> 1, y >> 1, z >> 1, lin);
        for (int h = 0; h < g.q; ++h)
        {
            double st[27];
            const double* fp = F.f[li - 1] + (long long)h * np;
#pragma unroll
            for (int o = 0; o < 27; ++o)
                st[o] = fp[lin[o]];
            F.f[li][(long long)h * n + i] = predict3(st, x & 1, y & 1, z & 1);
        }
        if (!ok)
            atomicAdd(&aux.err[0], 1);
    }
}

// ------------------------------------------------------------------ need mask + reconstruction
// need[li][c] = 1: the stream reads f^^ at cell c of level li.  Seeds (k3_need_seed): the
// 5^3 neighbourhood of every leaf at its own level (table stencils, gap-1 detail
// stencils) and, at the finest level, the one-cell shell around the leaf's finest box
// plus its boundary layer (E / A rims).  Propagation (k3_need_down, fine -> coarse): a
// needed cell outside the complete tree needs the 3^3 stencil of its parent.
__device__ __forceinline__ void mark_box3(const Geo3& g, int li, uint8_t* need, int x0, int x1, int y0, int y1, int z0,
                                          int z1)
{
    for (int x = x0; x <= x1; ++x)
        for (int y = y0; y <= y1; ++y)
            for (int z = z0; z <= z1; ++z)
                need[mr_lin3(g, li, x, y, z)] = 1;
}

// Table exactness of one (leaf, population, side), Decision D.13: dom_ok = every level-l
// dependency cell inside the domain (or periodic), par_ok = no parent of the touched
// level-(l+1) cells is internal
__device__ __forceinline__ void classify3(const Geo3& g, const Lv3& tn, const Tab3& tb, int li, int ti, int x, int y,
                                          int z, bool& dom_ok, bool& par_ok)
{
    const int* dep = tb.tdep + 6 * ti;
    dom_ok = true;
    if (!g.per[0])
        dom_ok = dom_ok && x + dep[0] >= 0 && x + dep[3] < g.nx[li];
    if (!g.per[1])
        dom_ok = dom_ok && y + dep[1] >= 0 && y + dep[4] < g.ny[li];
    if (!g.per[2])
        dom_ok = dom_ok && z + dep[2] >= 0 && z + dep[5] < g.nz[li];
    par_ok = true;
    if (dom_ok)
    {
        const int2 pr = tb.tpidx[ti];
        for (int k = 0; k < pr.y; ++k)
        {
            const int* o = tb.tpar + 3 * (pr.x + k);
            if (tn.kind[li][mr_lin3(g, li, x + o[0], y + o[1], z + o[2])] & K3_INT)
                par_ok = false;
        }
    }
}

// finest-level rim slab of the leaf box for an axis velocity: E of +e_a is the layer just
// below the box, A its last layer (mirrored for -e_a); returns the axis (-1: rest velocity)
__device__ __forceinline__ int rim_slab3(const int* eta, int side, int side_n, int x, int y, int z, int* lo, int* hi)
{
    lo[0] = x * side_n;
    lo[1] = y * side_n;
    lo[2] = z * side_n;
    for (int a = 0; a < 3; ++a)
        hi[a] = lo[a] + side_n;
    const int ax = eta[0] != 0 ? 0 : (eta[1] != 0 ? 1 : (eta[2] != 0 ? 2 : -1));
    if (ax >= 0)
    {
        const int e = eta[ax];
        const int c = side == 0 ? (e > 0 ? lo[ax] - 1 : hi[ax]) : (e > 0 ? hi[ax] - 1 : lo[ax]);
        lo[ax] = c;
        hi[ax] = c + 1;
    }
    return ax;
}

// WARP: one warp per cell of the level (coarse levels, rims of 4^gap finest cells): the
// lanes mark a slab together; else one thread per cell.
template <bool WARP>
__global__ void k3_need_seed(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 tn, const __grid_constant__ Bt3 need,
                             const Sch3* sc, const __grid_constant__ Tab3 tb, int li)
{
    const int lj = g.nlev - 1;
    const int gap = lj - li;
    const int* ud = tb.udep + 6 * gap;
    const int lane = threadIdx.x & 31;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long i = WARP ? tid >> 5 : tid; i < g.n[li]; i += WARP ? nth >> 5 : nth)
    {
        if (!(tn.kind[li][i] & K3_LEAF))
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        if (!WARP || lane == 0)
            mark_box3(g, li, need.b[li], x + ud[0], x + ud[3], y + ud[1], y + ud[4], z + ud[2], z + ud[5]);
        if (gap == 0)
            continue;
        for (int h = 0; h < g.q; ++h)
            for (int side = 0; side < 2; ++side)
            {
                bool dom_ok, par_ok;
                classify3(g, tn, tb, li, (gap * g.q + h) * 2 + side, x, y, z, dom_ok, par_ok);
                if (dom_ok && (par_ok || gap == 1))
                    continue;
                int lo[3], hi[3];
                if (rim_slab3(sc->eta[h], side, 1 << gap, x, y, z, lo, hi) < 0)
                    continue;
                if (!WARP)
                    mark_box3(g, lj, need.b[lj], lo[0], hi[0] - 1, lo[1], hi[1] - 1, lo[2], hi[2] - 1);
                else
                {
                    const int ny_ = hi[1] - lo[1], nz_ = hi[2] - lo[2];
                    const int total = (hi[0] - lo[0]) * ny_ * nz_;
                    for (int k = lane; k < total; k += 32)
                        need.b[lj][mr_lin3(g, lj, lo[0] + k / (nz_ * ny_), lo[1] + (k / nz_) % ny_, lo[2] + k % nz_)] = 1;
                }
            }
    }
}

__global__ void k3_need_down(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 tn, const __grid_constant__ Bt3 need,
                             int li)
{
    GS3(i, g.n[li])
    {
        if (!need.b[li][i] || tn.kind[li][i])
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        const int px = x >> 1, py = y >> 1, pz = z >> 1;
        mark_box3(g, li - 1, need.b[li - 1], px - 1, px + 1, py - 1, py + 1, pz - 1, pz + 1);
    }
}

// zero-detail reconstruction of the needed cells outside the complete tree, top-down
__global__ void __launch_bounds__(128) k3_recon(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 tn,
                                                const __grid_constant__ Bt3 need, const __grid_constant__ Fl3 F, int li)
{
    const long long n = g.n[li], np = g.n[li - 1];
    GS3(i, n)
    {
        if (tn.kind[li][i] || !need.b[li][i])
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        int lin[27];
        stencil_idx3(g, li - 1, nullptr, x >> 1, y >> 1, z >> 1, lin);
        for (int h = 0; h < g.q; ++h)
        {
            double st[27];
            const double* fp = F.f[li - 1] + (long long)h * np;
#pragma unroll
            for (int o = 0; o < 27; ++o)
                st[o] = fp[lin[o]];
            F.f[li][(long long)h * n + i] = predict3(st, x & 1, y & 1, z & 1);
        }
    }
}

// ------------------------------------------------------------------ K7/K8 stream + collide
__device__ __forceinline__ void equilibrium3(const Sch3* sc, int q, const double* m, double* meq)
{
    // MRLBM_EQ_ADVECTION_D3Q6: (u, Vx u, Vy u, Vz u, 0, 0)
    const double u = m[0];
    for (int i = 0; i < q; ++i)
        meq[i] = 0.0;
    meq[0] = u;
    meq[1] = __dmul_rn(sc->eqp[0], u);
    meq[2] = __dmul_rn(sc->eqp[1], u);
    meq[3] = __dmul_rn(sc->eqp[2], u);
}

// value of the complete leaf covering the finest cell (direct evaluation)
__device__ __forceinline__ double covering_leaf3(const Geo3& g, const Lv3& tn, const Fl3& F, int h, int cx, int cy, int cz,
                                                 int* err)
{
    for (int li = g.nlev - 1; li >= 0; --li)
    {
        const int sh = g.nlev - 1 - li;
        const long long lin = xyz2lin(g, li, cx >> sh, cy >> sh, cz >> sh);
        if (tn.kind[li][lin] & K3_LEAF)
            return F.f[li][(long long)h * g.n[li] + lin];
    }
    atomicAdd(&err[0], 1);
    return 0.0;
}

// One thread per leaf: per population the E / A sums by the flattened table when it is
// exact for this leaf (D.13), with the gap-1 detail correction (D.13b), else the sum over
// the finest rim cells of f^^ (boundary rule outside the domain); all
// sums serial from 0.0 in lexicographic order (D.12); then the MRT collision (D.24).
// MODE 1: one warp per cell of the level (coarse levels): the lanes fetch 32 rim cells at a
// time into shared memory and lane 0 accumulates them in the same serial order; every
// lane follows the same (leaf-uniform) control flow and lane 0 alone writes.
// MODE 2: one block of 2 q warps per cell (the coarsest levels, rims of >= 1024 cells): warp w
// takes the pair (population w / 2, side w % 2) the same way, thread 0 then assembles the
// populations from the 2 q sums and collides.  (With one warp per leaf the 12 pairs of a
// gap-5 leaf, 2 x 6 x 32 batches, were one dependent chain that set the duration of the
// level's launch.)
template <int MODE>
__global__ void __launch_bounds__(MODE == 2 ? 512 : 128) k3_stream_collide(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 tn,
                                                         const __grid_constant__ Fl3 Fin, const __grid_constant__ Fl3 Fout,
                                                         const Sch3* sc, const __grid_constant__ Tab3 tb, int li,
                                                         const __grid_constant__ Aux3 aux)
{
    const int q = g.q;
    const int lj = g.nlev - 1;
    const int gap = lj - li;
    const long long n = g.n[li], nf = g.n[lj];
    const int fx = g.nx[lj], fy = g.ny[lj], fz = g.nz[lj];
    const double scale = ldexp(1.0, 3 * (li - lj));
    const int side_n = 1 << gap;
    __shared__ double sv[MODE == 2 ? 16 : 4][32];
    __shared__ double ssum[32];
    __shared__ int sfb;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool writer = MODE == 0 || (MODE == 1 && lane == 0) || (MODE == 2 && threadIdx.x == 0);
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long i0 = MODE == 0 ? tid : (MODE == 1 ? tid >> 5 : blockIdx.x);
    const long long di = MODE == 0 ? nth : (MODE == 1 ? nth >> 5 : gridDim.x);
    for (long long i = i0; i < n; i += di)
    {
        if (!(tn.kind[li][i] & K3_LEAF))
            continue; // (block-uniform in MODE 2)
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        double f[kQ3];
        for (int h = 0; h < kQ3; ++h)
            f[h] = 0.0;
        bool any_fb = false;
        if (MODE == 2)
        {
            if (threadIdx.x == 0)
                sfb = 0;
            __syncthreads();
        }
        for (int h = 0; h < q; ++h)
        {
            if (MODE == 2 && h != (wid >> 1))
                continue;
            const double* fl = Fin.f[li] + (long long)h * n;
            const double* ff = Fin.f[lj] + (long long)h * nf;
            const double fstar = fl[i];
            double sums[2] = {0.0, 0.0};
            for (int side = 0; side < 2; ++side)
            {
                if (MODE == 2 && side != (wid & 1))
                    continue;
                const int ti = (gap * q + h) * 2 + side;
                const int2 tr = tb.tidx[ti];
                bool dom_ok, par_ok;
                classify3(g, tn, tb, li, ti, x, y, z, dom_ok, par_ok);
                double s = 0.0;
                int lo[3], hi[3];
                const int ax = rim_slab3(sc->eta[h], side, side_n, x, y, z, lo, hi);
                if (dom_ok && (par_ok || gap == 1))
                {
                    for (int k = 0; k < tr.y; ++k)
                    {
                        const int* o = tb.toff + 3 * (tr.x + k);
                        s = __dadd_rn(s, __dmul_rn(tb.tw[tr.x + k], fl[mr_lin3(g, li, x + o[0], y + o[1], z + o[2])]));
                    }
                    if (!par_ok && ax >= 0)
                    {
                        // gap 1 with finer neighbours: add the detail of every rim cell in the tree
                        any_fb = true;
                        for (int cx = lo[0]; cx < hi[0]; ++cx)
                            for (int cy = lo[1]; cy < hi[1]; ++cy)
                                for (int cz = lo[2]; cz < hi[2]; ++cz)
                                {
                                    const int wx = coord3(cx, fx, g.per[0]), wy = coord3(cy, fy, g.per[1]),
                                              wz = coord3(cz, fz, g.per[2]);
                                    const long long lin = xyz2lin(g, lj, wx, wy, wz);
                                    if (!tn.kind[lj][lin])
                                        continue;
                                    double st[27];
                                    load_stencil3(g, li, fl, nullptr, wx >> 1, wy >> 1, wz >> 1, st);
                                    s = __dadd_rn(s, __dsub_rn(ff[lin], predict3(st, wx & 1, wy & 1, wz & 1)));
                                }
                    }
                    else if (!par_ok)
                        any_fb = true;
                }
                else if (ax >= 0)
                {
                    any_fb = true;
                    // value of the finest rim cell: f^^ inside (E and A sides), boundary rule outside (E side)
                    auto rimval = [&](int cx, int cy, int cz) -> double {
                        int face = -1;
                        if (side == 0)
                        {
                            if (!g.per[0] && (cx < 0 || cx >= fx))
                                face = cx < 0 ? 0 : 1;
                            else if (!g.per[1] && (cy < 0 || cy >= fy))
                                face = cy < 0 ? 2 : 3;
                            else if (!g.per[2] && (cz < 0 || cz >= fz))
                                face = cz < 0 ? 4 : 5;
                        }
                        if (face < 0)
                            return ff[mr_lin3(g, lj, cx, cy, cz)];
                        const int kind = sc->bc_kind[face];
                        if (kind == MRLBM_BC_COPY)
                            return covering_leaf3(g, tn, Fin, h, coord3(cx, fx, g.per[0]), coord3(cy, fy, g.per[1]),
                                                  coord3(cz, fz, g.per[2]), aux.err);
                        const int hb = sc->opp[h];
                        if (hb < 0)
                        {
                            atomicAdd(&aux.err[2], 1);
                            return 0.0;
                        }
                        double v = Fin.f[li][(long long)hb * n + i];
                        if (kind == MRLBM_BC_ANTI_BOUNCE_BACK)
                            v = -v;
                        else if (kind == MRLBM_BC_VELOCITY_BOUNCE_BACK)
                            v = __dadd_rn(v, sc->bc_add[face][h]);
                        return v;
                    };
                    if (MODE == 0)
                    {
                        for (int cx = lo[0]; cx < hi[0]; ++cx)
                            for (int cy = lo[1]; cy < hi[1]; ++cy)
                                for (int cz = lo[2]; cz < hi[2]; ++cz)
                                    s = __dadd_rn(s, rimval(cx, cy, cz));
                    }
                    else
                    {
                        const int ny_ = hi[1] - lo[1], nz_ = hi[2] - lo[2];
                        const int total = (hi[0] - lo[0]) * ny_ * nz_;
                        for (int b0 = 0; b0 < total; b0 += 32)
                        {
                            const int k = b0 + lane;
                            sv[wid][lane] = k < total ? rimval(lo[0] + k / (nz_ * ny_), lo[1] + (k / nz_) % ny_, lo[2] + k % nz_) : 0.0;
                            __syncwarp();
                            if (lane == 0)
                            {
                                const int nv = min(32, total - b0);
                                for (int j = 0; j < nv; ++j)
                                    s = __dadd_rn(s, sv[wid][j]);
                            }
                            __syncwarp();
                        }
                    }
                }
                else
                    any_fb = any_fb || !(dom_ok && par_ok);
                sums[side] = s;
                if (MODE == 2 && lane == 0)
                    ssum[wid] = s;
            }
            if (MODE != 2)
                f[h] = __dadd_rn(fstar, __dmul_rn(scale, __dsub_rn(sums[0], sums[1])));
        }
        if (MODE == 2)
        {
            if (lane == 0 && any_fb)
                atomicOr(&sfb, 1);
            __syncthreads();
            if (threadIdx.x == 0)
            {
                for (int h = 0; h < q; ++h)
                    f[h] = __dadd_rn(Fin.f[li][(long long)h * n + i],
                                     __dmul_rn(scale, __dsub_rn(ssum[2 * h], ssum[2 * h + 1])));
                any_fb = sfb != 0;
            }
        }
        // collision: m = M f, m' = (1 - s) m + s m^eq, f* = M^-1 m' (DenseMatrix::multiply order)
        double m[kQ3], meq[kQ3], mp[kQ3];
        for (int r = 0; r < q; ++r)
        {
            double acc = 0.0;
            for (int c = 0; c < q; ++c)
                acc = __dadd_rn(acc, __dmul_rn(sc->M[r * q + c], f[c]));
            m[r] = acc;
        }
        equilibrium3(sc, q, m, meq);
        for (int r = 0; r < q; ++r)
            mp[r] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, sc->s[r]), m[r]), __dmul_rn(sc->s[r], meq[r]));
        bool finite = true;
        for (int r = 0; r < q; ++r)
        {
            double acc = 0.0;
            for (int c = 0; c < q; ++c)
                acc = __dadd_rn(acc, __dmul_rn(sc->Minv[r * q + c], mp[c]));
            finite = finite && isfinite(acc);
            if (writer)
                Fout.f[li][(long long)r * n + i] = acc;
        }
        if (writer && !finite)
            atomicAdd(&aux.err[1], 1);
        if (writer && any_fb)
            atomicAdd(&aux.cnt[2 * kL3], 1);
        if (MODE == 2)
            __syncthreads(); // ssum / sfb are reused by the block's next leaf
    }
}

// ------------------------------------------------------------------ load / read-back
__global__ void k3_load(const __grid_constant__ Geo3 g, int li, const int32_t* idx, const double* fin, long long nld,
                        uint8_t* kind, double* F, int* bad)
{
    GS3(i, nld)
    {
        const int x = idx[3 * i], y = idx[3 * i + 1], z = idx[3 * i + 2];
        if (x < 0 || x >= g.nx[li] || y < 0 || y >= g.ny[li] || z < 0 || z >= g.nz[li])
        {
            atomicAdd(bad, 1);
            continue;
        }
        const long long lin = xyz2lin(g, li, x, y, z);
        if (kind[lin])
            atomicAdd(bad, 1); // duplicate
        kind[lin] = K3_LEAF;
        for (int h = 0; h < g.q; ++h)
            F[(long long)h * g.n[li] + lin] = fin[(long long)h * nld + i];
    }
}

// ancestors of loaded leaves become internal nodes
__global__ void k3_load_up(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 t, int li)
{
    GS3(i, g.n[li])
    {
        if (!t.kind[li][i])
            continue;
        int x, y, z;
        lin2xyz(g, li, i, x, y, z);
        // byte read-modify-write: every writer ORs the same bit, so the race is benign
        uint8_t* p = t.kind[li - 1] + xyz2lin(g, li - 1, x >> 1, y >> 1, z >> 1);
        *p = *p | K3_INT;
    }
}

// the loaded leaves must form a complete-leaf partition: no leaf that is also internal,
// every child of an internal node (and every coarsest cell) present
__global__ void k3_load_check(const __grid_constant__ Geo3 g, const __grid_constant__ Lv3 t, int li, int* bad,
                              const __grid_constant__ Aux3 aux)
{
    __shared__ int sl, si;
    if (threadIdx.x == 0)
        sl = si = 0;
    __syncthreads();
    int nl = 0, ni = 0;
    GS3(i, g.n[li])
    {
        const uint8_t k = t.kind[li][i];
        if (k == (K3_LEAF | K3_INT))
            atomicAdd(bad, 1);
        bool inR = li == 0;
        if (!inR)
        {
            int x, y, z;
            lin2xyz(g, li, i, x, y, z);
            inR = (t.kind[li - 1][xyz2lin(g, li - 1, x >> 1, y >> 1, z >> 1)] & K3_INT) != 0;
        }
        if (inR != (k != 0))
            atomicAdd(bad, 1);
        if (li == g.nlev - 1 && (k & K3_INT))
            atomicAdd(bad, 1);
        nl += (k & K3_LEAF) != 0;
        ni += (k & K3_INT) != 0;
    }
    atomicAdd(&sl, nl);
    atomicAdd(&si, ni);
    __syncthreads();
    if (threadIdx.x == 0)
    {
        if (sl)
            atomicAdd(&aux.cnt[2 * li], sl);
        if (si)
            atomicAdd(&aux.cnt[2 * li + 1], si);
    }
}

// read-back compaction of the leaves of one level in lexicographic order: per-block
// counts, a single-block scan, then an ordered scatter (ballot ranks inside the block)
constexpr int kRB = 1024;
__global__ void __launch_bounds__(kRB) k3_rb_count(const uint8_t* kind, long long n, int* bc)
{
    __shared__ int s;
    if (threadIdx.x == 0)
        s = 0;
    __syncthreads();
    const long long i = (long long)blockIdx.x * kRB + threadIdx.x;
    const bool leaf = i < n && (kind[i] & K3_LEAF);
    const unsigned b = __ballot_sync(0xffffffffu, leaf);
    if ((threadIdx.x & 31) == 0 && b)
        atomicAdd(&s, __popc(b));
    __syncthreads();
    if (threadIdx.x == 0)
        bc[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) k3_rb_scan(int* bc, int nb)
{
    // exclusive scan of nb block counts by one block (chunks of 1024 with a carry)
    __shared__ int sh[1024];
    __shared__ int carry;
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024)
    {
        const int i = base + threadIdx.x;
        const int v = i < nb ? bc[i] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1)
        {
            const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < nb)
            bc[i] = carry + sh[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 0)
            carry += sh[1023];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kRB) k3_rb_scatter(const __grid_constant__ Geo3 g, int li, const uint8_t* kind,
                                                     const double* F, const int* bc, long long nleaf, int32_t* idx,
                                                     double* out)
{
    __shared__ int wsum[kRB / 32];
    const long long n = g.n[li];
    const long long i = (long long)blockIdx.x * kRB + threadIdx.x;
    const bool leaf = i < n && (kind[i] & K3_LEAF);
    const unsigned b = __ballot_sync(0xffffffffu, leaf);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
        wsum[w] = __popc(b);
    __syncthreads();
    if (!leaf)
        return;
    int off = bc[blockIdx.x];
    for (int k = 0; k < w; ++k)
        off += wsum[k];
    off += __popc(b & ((1u << lane) - 1u));
    int x, y, z;
    lin2xyz(g, li, i, x, y, z);
    if (idx)
    {
        idx[3 * (long long)off] = x;
        idx[3 * (long long)off + 1] = y;
        idx[3 * (long long)off + 2] = z;
    }
    if (out)
        for (int h = 0; h < g.q; ++h)
            out[(long long)h * nleaf + off] = F[(long long)h * n + i];
}

} // namespace

// ====================================================================== host side
struct Engine3D {
    mrlbm_scheme_spec sc{};
    mrlbm_run_config rc{};
    Geo3 geo{};
    cudaStream_t stream = nullptr;
    uint8_t* kind[2][kL3]{};
    double* F[2][kL3]{};
    uint8_t* keep[kL3]{};
    uint8_t* rn[kL3]{};
    uint8_t* need[kL3]{};
    Sch3* sch = nullptr;
    int2* tidx = nullptr;
    int* toff = nullptr;
    double* tw = nullptr;
    int* tdep = nullptr;
    int2* tpidx = nullptr;
    int* tpar = nullptr;
    int* udep = nullptr;
    int* err = nullptr;
    int* cnt = nullptr;
    int* bad = nullptr;
    int* rbc = nullptr;
    long long rbc_n = 0;
    mrlbm_tie_record* ties = nullptr;
    int* tie_n = nullptr;
    int* step_no = nullptr;
    int cur = 0;  // tree version
    int curf = 0; // buffer holding the state
    bool committed = false;
    long long ld_n[kL3]{};
    int64_t leaves[kL3]{}, internal[kL3]{};
    int64_t fallback = 0, leaf_updates = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long kcount = 0;
    std::string err_msg;
    int grid_cap = 148 * 16;
    int block_gap = kBlockGap3; // MRLBM_E3_BLOCK_GAP
    // MRLBM_E3_PROF=1: an event after every kernel of the step, totals printed at destroy
    bool prof = false;
    std::vector<cudaEvent_t> pev;
    std::vector<const char*> pname;
    std::vector<std::pair<std::string, double>> pacc;
    int psteps = 0;
};

namespace {

#define CU3(e, call)                                                                                           \
    do                                                                                                         \
    {                                                                                                          \
        cudaError_t _s = (call);                                                                               \
        if (_s != cudaSuccess)                                                                                 \
        {                                                                                                      \
            (e)->err_msg = std::string("CUDA error: ") + cudaGetErrorString(_s) + " at " #call;                \
            return MRLBM_ERR_CUDA;                                                                             \
        }                                                                                                      \
    } while (0)

int grid3(const Engine3D* e, long long n, int block)
{
    const long long b = (n + block - 1) / block;
    return (int)std::max(1LL, std::min<long long>(b, e->grid_cap));
}

Lv3 lv(const Engine3D* e, int v)
{
    Lv3 t{};
    for (int i = 0; i < kL3; ++i)
        t.kind[i] = e->kind[v][i];
    return t;
}
Fl3 fl(const Engine3D* e, int b)
{
    Fl3 t{};
    for (int i = 0; i < kL3; ++i)
        t.f[i] = e->F[b][i];
    return t;
}
Bt3 bt(uint8_t* const* p)
{
    Bt3 t{};
    for (int i = 0; i < kL3; ++i)
        t.b[i] = p[i];
    return t;
}
Aux3 aux3(const Engine3D* e)
{
    Aux3 a{};
    a.err = e->err;
    a.cnt = e->cnt;
    a.ties = e->ties;
    a.tie_n = e->tie_n;
    a.step_no = e->step_no;
    return a;
}
Tab3 tab3(const Engine3D* e)
{
    Tab3 t{};
    t.tidx = e->tidx;
    t.toff = e->toff;
    t.tw = e->tw;
    t.tdep = e->tdep;
    t.tpidx = e->tpidx;
    t.tpar = e->tpar;
    t.udep = e->udep;
    return t;
}

int read_counts(Engine3D* e)
{
    int h[2 * kL3 + 1];
    CU3(e, cudaMemcpyAsync(h, e->cnt, sizeof(h), cudaMemcpyDeviceToHost, e->stream));
    CU3(e, cudaStreamSynchronize(e->stream));
    for (int li = 0; li < e->geo.nlev; ++li)
    {
        e->leaves[li] = h[2 * li];
        e->internal[li] = h[2 * li + 1];
    }
    e->fallback = h[2 * kL3];
    return MRLBM_OK;
}

int check_err(Engine3D* e)
{
    int h[4];
    CU3(e, cudaMemcpyAsync(h, e->err, sizeof(h), cudaMemcpyDeviceToHost, e->stream));
    CU3(e, cudaStreamSynchronize(e->stream));
    if (h[2])
    {
        e->err_msg = "bounce-back needs an opposite velocity";
        return MRLBM_ERR_CONFIG;
    }
    if (h[0])
    {
        e->err_msg = "mesh invariant violated: unresolved prediction stencil (grading)";
        return MRLBM_ERR_CAPACITY;
    }
    if (h[1])
    {
        e->err_msg = "non-finite population after collision";
        return MRLBM_ERR_NUMERIC;
    }
    return MRLBM_OK;
}

void pmark(Engine3D* e, const char* name)
{
    ++e->kcount;
    if (!e->prof)
        return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, e->stream);
    e->pev.push_back(ev);
    e->pname.push_back(name);
}

void pflush(Engine3D* e)
{
    if (!e->prof || e->pev.empty())
        return;
    cudaStreamSynchronize(e->stream);
    for (size_t k = 1; k < e->pev.size(); ++k)
    {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e->pev[k - 1], e->pev[k]);
        bool found = false;
        for (auto& a : e->pacc)
            if (a.first == e->pname[k])
            {
                a.second += ms;
                found = true;
            }
        if (!found)
            e->pacc.emplace_back(e->pname[k], ms);
    }
    for (auto ev : e->pev)
        cudaEventDestroy(ev);
    e->pev.clear();
    e->pname.clear();
    ++e->psteps;
}

int one_step(Engine3D* e)
{
    const Geo3& g = e->geo;
    const int nl = g.nlev;
    cudaStream_t s = e->stream;
    const int vo = e->cur, vn = e->cur ^ 1;
    const int bi = e->curf, bo = e->curf ^ 1;
    const Lv3 to = lv(e, vo), tn = lv(e, vn);
    const Fl3 Fi = fl(e, bi), Fo = fl(e, bo);
    const Bt3 keep = bt(e->keep), rn = bt(e->rn), need = bt(e->need);
    const Aux3 aux = aux3(e);
    const Tab3 tb = tab3(e);
    for (int li = 0; li < nl; ++li)
    {
        CU3(e, cudaMemsetAsync(e->keep[li], 0, g.n[li], s));
        CU3(e, cudaMemsetAsync(e->rn[li], 0, g.n[li], s));
        CU3(e, cudaMemsetAsync(e->need[li], 0, g.n[li], s));
    }
    CU3(e, cudaMemsetAsync(e->cnt, 0, sizeof(int) * (2 * kL3 + 1), s));
    pmark(e, "memset");
    // K1: projection of the old tree, fine -> coarse
    for (int li = nl - 2; li >= 0; --li)
    {
        k3_project<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, to, Fi, li);
        pmark(e, "k3_project");
    }
    // K2: details, group flags
    for (int li = 0; li < nl - 1; ++li)
    {
        k3_details<<<grid3(e, g.n[li], 128), 128, 0, s>>>(g, to, Fi, keep, rn, e->sch, li, aux);
        pmark(e, "k3_details");
    }
    // K3: closure, enlargement, grading
    for (int li = nl - 2; li >= 1; --li)
    {
        k3_closure<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, keep, li);
        pmark(e, "k3_closure");
    }
    for (int li = 0; li < nl - 1; ++li)
    {
        k3_enlarge<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, keep, rn, e->sch, li);
        pmark(e, "k3_enlarge");
    }
    for (int li = nl - 2; li >= 1; --li)
    {
        k3_grade<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, rn, li);
        pmark(e, "k3_grade");
    }
    // K4: the new tree
    for (int li = 0; li < nl; ++li)
    {
        k3_kinds<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, rn, tn, li, aux);
        pmark(e, "k3_kinds");
    }
    // K5: transfer, coarse -> fine; K6: projection of the new tree
    for (int li = 1; li < nl; ++li)
    {
        k3_transfer<<<grid3(e, g.n[li], 128), 128, 0, s>>>(g, to, tn, Fi, li, aux);
        pmark(e, "k3_transfer");
    }
    for (int li = nl - 2; li >= 0; --li)
    {
        k3_project<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, tn, Fi, li);
        pmark(e, "k3_project");
    }
    // need mask and zero-detail reconstruction of the cells the stream reads
    for (int li = 0; li < nl; ++li)
    {
        if (nl - 1 - li >= kWarpGap3)
            k3_need_seed<true><<<grid3(e, g.n[li] * 32, 256), 256, 0, s>>>(g, tn, need, e->sch, tb, li);
        else
            k3_need_seed<false><<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, tn, need, e->sch, tb, li);
        pmark(e, "k3_need_seed");
    }
    for (int li = nl - 1; li >= 1; --li)
    {
        k3_need_down<<<grid3(e, g.n[li], 256), 256, 0, s>>>(g, tn, need, li);
        pmark(e, "k3_need_down");
    }
    for (int li = 1; li < nl; ++li)
    {
        k3_recon<<<grid3(e, g.n[li], 128), 128, 0, s>>>(g, tn, need, Fi, li);
        pmark(e, "k3_recon");
    }
    // K7 / K8: stream + collide
    for (int li = 0; li < nl; ++li)
    {
        if (nl - 1 - li >= e->block_gap)
            k3_stream_collide<2><<<(int)std::min<long long>(g.n[li], e->grid_cap), 64 * g.q, 0, s>>>(g, tn, Fi, Fo, e->sch, tb, li, aux);
        else if (nl - 1 - li >= kWarpGap3)
            k3_stream_collide<1><<<grid3(e, g.n[li] * 32, 128), 128, 0, s>>>(g, tn, Fi, Fo, e->sch, tb, li, aux);
        else
            k3_stream_collide<0><<<grid3(e, g.n[li], 128), 128, 0, s>>>(g, tn, Fi, Fo, e->sch, tb, li, aux);
        pmark(e, "k3_stream_collide");
    }
    e->cur = vn;
    e->curf = bo;
    pflush(e);
    CU3(e, cudaGetLastError());
    return MRLBM_OK;
}

__global__ void k3_inc(int* p)
{
    *p += 1;
}

} // namespace

int e3_create(const mrlbm_scheme_spec* sc, const mrlbm_run_config* rc, Engine3D** out, std::string& err)
{
    *out = nullptr;
    if (sc->d != 3 || sc->q < 1 || sc->q > kQ3 || sc->equilibrium != MRLBM_EQ_ADVECTION_D3Q6 || sc->q != 6)
    {
        err = "3D path: only the D3Q6 advection scheme (q = 6, MRLBM_EQ_ADVECTION_D3Q6) is built";
        return MRLBM_ERR_CONFIG;
    }
    if (rc->j_min < 0 || rc->j_max <= rc->j_min || rc->j_max - rc->j_min + 1 > kL3 || rc->gamma != 1 ||
        rc->graduation != 1 || sc->nblocks != 1 || rc->obstacle != 0)
    {
        err = "3D path: bad run configuration";
        return MRLBM_ERR_CONFIG;
    }
    for (int h = 0; h < sc->q; ++h)
    {
        int nz = 0;
        for (int a = 0; a < 3; ++a)
        {
            if (std::abs(sc->eta[h][a]) > 1)
                nz = 9;
            nz += sc->eta[h][a] != 0;
        }
        if (nz > 1)
        {
            err = "3D path: velocities must be axis aligned with |eta_i| <= 1";
            return MRLBM_ERR_CONFIG;
        }
    }
    for (int a = 0; a < 3; ++a)
        if ((rc->bc_kind[2 * a] == MRLBM_BC_PERIODIC) != (rc->bc_kind[2 * a + 1] == MRLBM_BC_PERIODIC) ||
            rc->base_cells[a] < 1)
        {
            err = "3D path: bad domain / boundary configuration";
            return MRLBM_ERR_CONFIG;
        }
    Engine3D* e = new Engine3D();
    e->prof = std::getenv("MRLBM_E3_PROF") != nullptr;
    if (const char* bg = std::getenv("MRLBM_E3_BLOCK_GAP"))
        e->block_gap = std::max(2, std::atoi(bg));
    e->sc = *sc;
    e->rc = *rc;
    Geo3& g = e->geo;
    g.J0 = rc->j_min;
    g.J1 = rc->j_max;
    g.nlev = g.J1 - g.J0 + 1;
    g.q = sc->q;
    for (int a = 0; a < 3; ++a)
        g.per[a] = rc->bc_kind[2 * a] == MRLBM_BC_PERIODIC;
    long long total = 0;
    for (int li = 0; li < g.nlev; ++li)
    {
        const long long nx = rc->base_cells[0] << li, ny = rc->base_cells[1] << li, nz = rc->base_cells[2] << li;
        if (nx * ny * nz >= (1LL << 31))
        {
            delete e;
            err = "3D path: level box exceeds 2^31 cells";
            return MRLBM_ERR_CONFIG;
        }
        g.nx[li] = (int)nx;
        g.ny[li] = (int)ny;
        g.nz[li] = (int)nz;
        g.n[li] = nx * ny * nz;
        total += g.n[li];
    }
    auto fail = [&](const char* what) {
        err = std::string("3D path: ") + what + ": " + cudaGetErrorString(cudaGetLastError());
        e3_destroy(e);
        return MRLBM_ERR_CUDA;
    };
    if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail("stream");
    cudaEventCreate(&e->ev0);
    cudaEventCreate(&e->ev1);
    for (int li = 0; li < g.nlev; ++li)
    {
        // byte arrays padded to a multiple of 4 (k3_load_up ORs aligned words)
        const size_t nb = (size_t)((g.n[li] + 3) & ~3LL);
        for (int v = 0; v < 2; ++v)
        {
            if (cudaMalloc(&e->kind[v][li], nb) != cudaSuccess || cudaMemset(e->kind[v][li], 0, nb) != cudaSuccess)
                return fail("kind");
            if (cudaMalloc(&e->F[v][li], sizeof(double) * g.q * g.n[li]) != cudaSuccess ||
                cudaMemset(e->F[v][li], 0, sizeof(double) * g.q * g.n[li]) != cudaSuccess)
                return fail("fields");
        }
        if (cudaMalloc(&e->keep[li], nb) != cudaSuccess || cudaMalloc(&e->rn[li], nb) != cudaSuccess ||
            cudaMalloc(&e->need[li], nb) != cudaSuccess)
            return fail("flags");
    }
    // scheme constants
    Sch3 hs{};
    for (int h = 0; h < g.q; ++h)
    {
        for (int a = 0; a < 3; ++a)
            hs.eta[h][a] = sc->eta[h][a];
        hs.opp[h] = -1;
        for (int k = 0; k < g.q; ++k)
            if (sc->eta[k][0] == -sc->eta[h][0] && sc->eta[k][1] == -sc->eta[h][1] && sc->eta[k][2] == -sc->eta[h][2])
            {
                hs.opp[h] = k;
                break;
            }
        hs.s[h] = sc->s[h];
    }
    std::memcpy(hs.M, sc->M, sizeof(double) * g.q * g.q);
    std::memcpy(hs.Minv, sc->Minv, sizeof(double) * g.q * g.q);
    std::memcpy(hs.eqp, sc->eq_params, sizeof(hs.eqp));
    hs.equilibrium = sc->equilibrium;
    for (int f = 0; f < 6; ++f)
    {
        hs.bc_kind[f] = rc->bc_kind[f];
        for (int h = 0; h < g.q; ++h)
            hs.bc_add[f][h] = rc->bc_add[f][h];
    }
    hs.eps = rc->epsilon;
    hs.mu = rc->mu;
    if (cudaMalloc(&e->sch, sizeof(Sch3)) != cudaSuccess ||
        cudaMemcpy(e->sch, &hs, sizeof(Sch3), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail("scheme");
    // flattened tables for every gap
    std::vector<int2> tidx, tpidx;
    std::vector<int> toff, tdep, tpar, udep;
    std::vector<double> tw;
    for (int gp = 0; gp < g.nlev; ++gp)
    {
        // union of the dependency boxes of the gap; gap 1 also covers the 5^3 box of the
        // detail-correction stencils (D.13b)
        int ulo[3] = {0, 0, 0}, uhi[3] = {0, 0, 0};
        if (gp == 1)
            for (int a = 0; a < 3; ++a)
            {
                ulo[a] = -2;
                uhi[a] = 2;
            }
        for (int h = 0; h < g.q; ++h)
            for (int side = 0; side < 2; ++side)
            {
                std::vector<TableEntry3> t;
                TableSets3 ts{};
                if (build_stream_table3(gp, sc->eta[h], side, t, &ts) != MRLBM_OK)
                {
                    err = "3D path: table construction failed";
                    e3_destroy(e);
                    return MRLBM_ERR_CONFIG;
                }
                tidx.push_back(make_int2((int)tw.size(), (int)t.size()));
                for (const auto& en : t)
                {
                    toff.insert(toff.end(), en.off, en.off + 3);
                    tw.push_back(en.w);
                }
                tdep.insert(tdep.end(), ts.dep_lo, ts.dep_lo + 3);
                tdep.insert(tdep.end(), ts.dep_hi, ts.dep_hi + 3);
                for (int a = 0; a < 3; ++a)
                {
                    ulo[a] = std::min(ulo[a], ts.dep_lo[a]);
                    uhi[a] = std::max(uhi[a], ts.dep_hi[a]);
                    for (const auto& en : t)
                    {
                        ulo[a] = std::min(ulo[a], en.off[a]);
                        uhi[a] = std::max(uhi[a], en.off[a]);
                    }
                }
                tpidx.push_back(make_int2((int)tpar.size() / 3, (int)ts.par.size()));
                for (const auto& p : ts.par)
                    tpar.insert(tpar.end(), p.begin(), p.end());
            }
        udep.insert(udep.end(), ulo, ulo + 3);
        udep.insert(udep.end(), uhi, uhi + 3);
    }
    auto up = [&](auto** dptr, const auto& v) {
        using T = std::remove_reference_t<decltype(v[0])>;
        const size_t bytes = sizeof(T) * std::max<size_t>(1, v.size());
        if (cudaMalloc(dptr, bytes) != cudaSuccess)
            return false;
        return v.empty() || cudaMemcpy(*dptr, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up(&e->tidx, tidx) || !up(&e->toff, toff) || !up(&e->tw, tw) || !up(&e->tdep, tdep) || !up(&e->tpidx, tpidx) ||
        !up(&e->tpar, tpar) || !up(&e->udep, udep))
        return fail("tables");
    e->rbc_n = (g.n[g.nlev - 1] + kRB - 1) / kRB;
    if (cudaMalloc(&e->err, sizeof(int) * 4) != cudaSuccess || cudaMemset(e->err, 0, sizeof(int) * 4) != cudaSuccess ||
        cudaMalloc(&e->cnt, sizeof(int) * (2 * kL3 + 1)) != cudaSuccess ||
        cudaMemset(e->cnt, 0, sizeof(int) * (2 * kL3 + 1)) != cudaSuccess ||
        cudaMalloc(&e->bad, sizeof(int)) != cudaSuccess || cudaMemset(e->bad, 0, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&e->rbc, sizeof(int) * e->rbc_n) != cudaSuccess ||
        cudaMalloc(&e->ties, sizeof(mrlbm_tie_record) * kTieCap3) != cudaSuccess ||
        cudaMalloc(&e->tie_n, sizeof(int)) != cudaSuccess || cudaMemset(e->tie_n, 0, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&e->step_no, sizeof(int)) != cudaSuccess || cudaMemset(e->step_no, 0, sizeof(int)) != cudaSuccess)
        return fail("aux");
    *out = e;
    return MRLBM_OK;
}

int e3_load_leaves(Engine3D* e, int level, int64_t n, const int32_t* idx, const double* f)
{
    const Geo3& g = e->geo;
    if (level < g.J0 || level > g.J1 || n < 0 || (n > 0 && (!idx || !f)))
    {
        e->err_msg = "load: level out of range or null buffers";
        return MRLBM_ERR_CONFIG;
    }
    const int li = level - g.J0;
    // first load after create / commit: start from an empty tree
    bool fresh = true;
    for (int k = 0; k < g.nlev; ++k)
        fresh = fresh && e->ld_n[k] == 0;
    if (fresh)
    {
        e->cur = 0;
        e->curf = 0;
        for (int k = 0; k < g.nlev; ++k)
            CU3(e, cudaMemsetAsync(e->kind[0][k], 0, (size_t)((g.n[k] + 3) & ~3LL), e->stream));
        CU3(e, cudaMemsetAsync(e->bad, 0, sizeof(int), e->stream));
        e->committed = false;
    }
    if (n == 0)
        return MRLBM_OK;
    if (n > g.n[li])
    {
        e->err_msg = "load: more leaves than cells at this level";
        return MRLBM_ERR_CONFIG;
    }
    int32_t* didx = nullptr;
    double* df = nullptr;
    CU3(e, cudaMalloc(&didx, sizeof(int32_t) * 3 * n));
    CU3(e, cudaMalloc(&df, sizeof(double) * g.q * n));
    CU3(e, cudaMemcpyAsync(didx, idx, sizeof(int32_t) * 3 * n, cudaMemcpyHostToDevice, e->stream));
    CU3(e, cudaMemcpyAsync(df, f, sizeof(double) * g.q * n, cudaMemcpyHostToDevice, e->stream));
    k3_load<<<grid3(e, n, 256), 256, 0, e->stream>>>(g, li, didx, df, n, e->kind[0][li], e->F[0][li], e->bad);
    ++e->kcount;
    CU3(e, cudaStreamSynchronize(e->stream));
    cudaFree(didx);
    cudaFree(df);
    e->ld_n[li] += n;
    return MRLBM_OK;
}

int e3_commit(Engine3D* e)
{
    const Geo3& g = e->geo;
    const Lv3 t = lv(e, 0);
    const Aux3 aux = aux3(e);
    for (int li = g.nlev - 1; li >= 1; --li)
    {
        k3_load_up<<<grid3(e, g.n[li], 256), 256, 0, e->stream>>>(g, t, li);
        ++e->kcount;
    }
    CU3(e, cudaMemsetAsync(e->cnt, 0, sizeof(int) * (2 * kL3 + 1), e->stream));
    for (int li = 0; li < g.nlev; ++li)
    {
        k3_load_check<<<grid3(e, g.n[li], 256), 256, 0, e->stream>>>(g, t, li, e->bad, aux);
        ++e->kcount;
    }
    int bad = 0;
    CU3(e, cudaMemcpyAsync(&bad, e->bad, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    CU3(e, cudaStreamSynchronize(e->stream));
    for (int li = 0; li < g.nlev; ++li)
        e->ld_n[li] = 0;
    if (bad)
    {
        e->err_msg = "load: leaves do not form a complete-leaf partition of the domain";
        return MRLBM_ERR_CONFIG;
    }
    const int st = read_counts(e);
    if (st != MRLBM_OK)
        return st;
    CU3(e, cudaMemsetAsync(e->err, 0, sizeof(int) * 4, e->stream));
    CU3(e, cudaMemsetAsync(e->tie_n, 0, sizeof(int), e->stream));
    CU3(e, cudaMemsetAsync(e->step_no, 0, sizeof(int), e->stream));
    e->cur = 0;
    e->curf = 0;
    e->committed = true;
    e->leaf_updates = 0;
    return MRLBM_OK;
}

int e3_step(Engine3D* e, int nsteps, mrlbm_step_stats* stats)
{
    if (!e->committed)
    {
        e->err_msg = "step before commit";
        return MRLBM_ERR_STATE;
    }
    const Geo3& g = e->geo;
    const long long k0 = e->kcount;
    CU3(e, cudaEventRecord(e->ev0, e->stream));
    int status = MRLBM_OK;
    for (int it = 0; it < nsteps; ++it)
    {
        status = one_step(e);
        if (status != MRLBM_OK)
            break;
        k3_inc<<<1, 1, 0, e->stream>>>(e->step_no);
        ++e->kcount;
        // one host sync per step: error flags and level counts
        status = check_err(e);
        if (status != MRLBM_OK)
            break;
        status = read_counts(e);
        if (status != MRLBM_OK)
            break;
        for (int li = 0; li < g.nlev; ++li)
            e->leaf_updates += e->leaves[li];
    }
    CU3(e, cudaEventRecord(e->ev1, e->stream));
    CU3(e, cudaEventSynchronize(e->ev1));
    if (stats)
    {
        std::memset(stats, 0, sizeof(*stats));
        stats->levels = g.nlev;
        for (int li = 0; li < g.nlev; ++li)
        {
            stats->leaves[li] = e->leaves[li];
            stats->internal[li] = e->internal[li];
        }
        stats->fallback_leaves = e->fallback;
        stats->leaf_updates = e->leaf_updates;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e->ev0, e->ev1);
        stats->ms_total = ms;
        stats->kernel_launches = e->kcount - k0;
        int64_t ns = 0, ni = 0;
        for (int li = 0; li < g.nlev; ++li)
        {
            ns += e->leaves[li];
            ni += e->internal[li];
        }
        // SURVEY 8d model with old ~ new counts: 8 q (7 N_S + 4 N_I)
        stats->bytes_model = 8LL * g.q * (7 * ns + 4 * ni);
        stats->bytes_stream = 8LL * g.q * 2 * ns;
    }
    if (status != MRLBM_OK)
        e->committed = false;
    return status;
}

int e3_level_count(Engine3D* e, int level, int64_t* n)
{
    const Geo3& g = e->geo;
    if (level < g.J0 || level > g.J1 || !n)
        return MRLBM_ERR_CONFIG;
    *n = e->leaves[level - g.J0];
    return MRLBM_OK;
}

int e3_read_leaves(Engine3D* e, int level, int32_t* idx, double* f)
{
    const Geo3& g = e->geo;
    if (level < g.J0 || level > g.J1)
        return MRLBM_ERR_CONFIG;
    const int li = level - g.J0;
    const long long nleaf = e->leaves[li];
    if (nleaf == 0)
        return MRLBM_OK;
    const int nb = (int)((g.n[li] + kRB - 1) / kRB);
    int32_t* didx = nullptr;
    double* df = nullptr;
    if (idx)
        CU3(e, cudaMalloc(&didx, sizeof(int32_t) * 3 * nleaf));
    if (f)
        CU3(e, cudaMalloc(&df, sizeof(double) * g.q * nleaf));
    k3_rb_count<<<nb, kRB, 0, e->stream>>>(e->kind[e->cur][li], g.n[li], e->rbc);
    k3_rb_scan<<<1, 1024, 0, e->stream>>>(e->rbc, nb);
    k3_rb_scatter<<<nb, kRB, 0, e->stream>>>(g, li, e->kind[e->cur][li], e->F[e->curf][li], e->rbc, nleaf, didx, df);
    e->kcount += 3;
    if (idx)
        CU3(e, cudaMemcpyAsync(idx, didx, sizeof(int32_t) * 3 * nleaf, cudaMemcpyDeviceToHost, e->stream));
    if (f)
        CU3(e, cudaMemcpyAsync(f, df, sizeof(double) * g.q * nleaf, cudaMemcpyDeviceToHost, e->stream));
    CU3(e, cudaStreamSynchronize(e->stream));
    cudaFree(didx);
    cudaFree(df);
    return MRLBM_OK;
}

int e3_tie_log(Engine3D* e, mrlbm_tie_record* out, int cap, int64_t* n, int reset)
{
    int k = 0;
    CU3(e, cudaMemcpyAsync(&k, e->tie_n, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    CU3(e, cudaStreamSynchronize(e->stream));
    if (n)
        *n = k;
    const int have = std::min(k, kTieCap3);
    std::vector<mrlbm_tie_record> h(have);
    if (have)
        CU3(e, cudaMemcpy(h.data(), e->ties, sizeof(mrlbm_tie_record) * have, cudaMemcpyDeviceToHost));
    std::sort(h.begin(), h.end(), [](const mrlbm_tie_record& a, const mrlbm_tie_record& b) {
        if (a.step != b.step) return a.step < b.step;
        if (a.level != b.level) return a.level < b.level;
        for (int i = 0; i < 3; ++i)
            if (a.cell[i] != b.cell[i]) return a.cell[i] < b.cell[i];
        return a.which < b.which;
    });
    for (int i = 0; out && i < cap && i < have; ++i)
        out[i] = h[i];
    if (reset)
        CU3(e, cudaMemsetAsync(e->tie_n, 0, sizeof(int), e->stream));
    if (k > kTieCap3)
    {
        e->err_msg = "tie log overflow";
        return MRLBM_ERR_CAPACITY;
    }
    return MRLBM_OK;
}

int e3_finest_count(const Engine3D* e, int64_t* n)
{
    *n = e->geo.n[e->geo.nlev - 1];
    return MRLBM_OK;
}

void* e3_stream(Engine3D* e)
{
    return static_cast<void*>(e->stream);
}

int e3_synchronize(Engine3D* e)
{
    CU3(e, cudaStreamSynchronize(e->stream));
    return MRLBM_OK;
}

const char* e3_last_error(const Engine3D* e)
{
    return e->err_msg.c_str();
}

void e3_destroy(Engine3D* e)
{
    if (!e)
        return;
    if (e->stream)
        cudaStreamSynchronize(e->stream);
    if (e->prof && e->psteps)
        for (const auto& a : e->pacc)
            std::fprintf(stderr, "e3prof %-20s %9.1f us/step\n", a.first.c_str(), 1e3 * a.second / e->psteps);
    for (int li = 0; li < kL3; ++li)
    {
        for (int v = 0; v < 2; ++v)
        {
            cudaFree(e->kind[v][li]);
            cudaFree(e->F[v][li]);
        }
        cudaFree(e->keep[li]);
        cudaFree(e->rn[li]);
        cudaFree(e->need[li]);
    }
    cudaFree(e->sch);
    cudaFree(e->tidx);
    cudaFree(e->toff);
    cudaFree(e->tw);
    cudaFree(e->tdep);
    cudaFree(e->tpidx);
    cudaFree(e->tpar);
    cudaFree(e->udep);
    cudaFree(e->err);
    cudaFree(e->cnt);
    cudaFree(e->bad);
    cudaFree(e->rbc);
    cudaFree(e->ties);
    cudaFree(e->tie_n);
    cudaFree(e->step_no);
    if (e->ev0)
        cudaEventDestroy(e->ev0);
    if (e->ev1)
        cudaEventDestroy(e->ev1);
    if (e->stream)
        cudaStreamDestroy(e->stream);
    delete e;
}

} // namespace mrlbm_b200
