// mrlbm_step.cu — B200 (sm_100a) implementation of one adaptive MR-LBM time step
// (Algorithm 1 body) behind the C-ABI in include/mrlbm_gpu.h.
//
// Data layout in HBM, per level m:
//   kind2[v][m] uint8 dense over the level box: leaf / internal / virtual (+ fallback)
//               of tree version v (old and new trees alternate)
//   cells[v][m] int32 slot -> linear cell index (row-major, last axis fastest);
//               slots: leaves [0,nL) | internal [nL,nL+nI) | virtual [.., +nV),
//               each range in lexicographic order == reference CellIndex order
//               (cell_set.hpp:333-354); used for iteration and read-back order
//   F[0/1][m]   fp64 values DENSE over the level box, one contiguous array per
//               population (index h*cells + linear index): stencil reads are direct
//               row-coalesced loads, no index lookups.  F[curf] is the state f*;
//               the transfer is done in place in it and the stream writes the other
//               buffer, which becomes the next state.
//   rn/keep/fbm/fbd dense per-step scratch flags
// Arithmetic mirrors the reference operation order exactly (no FMA: --fmad=false):
//   project  prediction.hpp:51-60     predict dense_matrix.hpp:42-54 (matvec)
//   predict  prediction.hpp:143-173   (center + s0 qx + s1 qy - s0 s1 qxy)
// so meshes and fields are bit-identical to the CPU oracle.
#include "mrlbm_internal.h"

#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

namespace mrlbm_b200 {

namespace cg = cooperative_groups;

constexpr int kL = MRLBM_MAX_LEVELS;
constexpr int kQ = MRLBM_MAX_Q;

enum : uint8_t { K_LEAF = 1, K_INT = 2, K_VIRT = 4, K_FB = 8, K_FBC = 16 };
// fallback leaves with gap >= kDeepGap stream in the dedicated K8 kernel (long
// serial rims, 2Q-way parallel per leaf); shallower ones inline in K7
constexpr int kDeepGap = 1;

struct Geo {
    int d, q, J0, J1, nlev, per0, per1;
    int nx[kL], ny[kL];
    int lny[kL]; // log2(ny) when ny is a power of two, else -1
    long long cap[kL];
};

struct Tree {
    uint8_t* kind[kL];  // dense per cell: K_LEAF / K_INT / K_VIRT (+ K_FB) of this tree version
    int32_t* cells[kL]; // slot -> linear index: leaves | internal | virtual, each lexicographic
    uint8_t* skind[kL]; // slot -> kind of that cell (read with cells[], no dependent gather)
    int* cnt;           // [nlev][4] = nL, nI, nV, -
};

struct Fld {
    double* f[kL];
};

struct Flags {
    uint8_t* kind[kL];
    uint8_t* rn[kL];
    uint8_t* keep[kL];
    unsigned* fbm[kL]; // dense per cell: invalid (population, side) mask of fallback leaves
    unsigned* fbd[kL]; // dense per cell: pairs whose dependencies leave the domain
};

struct SchemeDev {
    int q, nblocks, bs, eq, mu, obstacle, obs_ns;
    double lambda, eps;
    int eta[kQ][2];
    int opp[kQ];
    double M[kQ * kQ], Minv[kQ * kQ], s[kQ], eqp[8];
    int bc_kind[4];
    double bc_add[4][kQ];
    double origin[2], obs_c[2], obs_r, obs_feq[kQ];
};

struct Aux {
    int* err;          // [0] unresolved stencil, [1] non-finite, [2] inconsistency
    int* fb_count;     // fallback leaves of the current step
    int2* fb_list;     // (level, lin)
    unsigned* fb_mask; // per fallback leaf: bit (2h + side) set = table not exact
    unsigned* fb_dmask; // per fallback leaf: bit set = dependency leaves the domain
    long long fb_cap;
    long long* updates; // accumulated leaf updates
    const int2* tidx;   // [(g * q + h) * 2 + side] -> (start, count)
    const int2* toff;
    const double* tw;
    const int4* tdep;   // [(g * q + h) * 2 + side] -> dependency box (xlo, xhi, ylo, yhi)
    const int2* tpidx;  // [(g * q + h) * 2 + side] -> (start, count) into tpar
    const int2* tpar;   // parents of the level-(l+1) funnel
    const int2* guidx;  // [g] -> (start, count) into guoff: distinct table offsets of the gap
    const int2* guoff;
    const uint8_t* tu;  // per table entry: index into its gap's distinct offsets
    const int4* udep;   // [g] union of the dependency boxes
    const int2* upidx;  // [g] -> (start, count) into upar
    const int2* upar;   // [g] union of the parent sets
    const int2* eta;    // [h] logical velocities (x, y)
    const unsigned short* pmask; // [(g * q + h) * 2 + side] parents as bits of the 3^d box ((ox+1)*3+(oy+1))
    const unsigned short* umask; // [g] union over the pairs
    // obstacle force tracking (null when off): per level, a dense box over the disc's
    // bounding box holding each leaf's (Fx, Fy) term of the current step
    int k8_long;        // > 0: leaves with gap >= k8_long (long rims) take the warp-cooperative K8 launch
    int fb1t;           // thread-per-leaf gap-1 path on: the boundary-rim fallback leaves are listed
    int* fbs;           // [2] segment lists of linear indices: 0 = gap-0 fallback leaves (level J1),
                        //     1 = gap-1 fallback leaves with domain-leaving pairs (level J1-1);
                        //     2 = the other gap-1 fallback leaves (level J1-1, K7 MODE 2),
                        //     counts at fb_count[2 + seg]
    long long fbs_off[3], fbs_cap[3];
    double* frc;
    // obstacle volume fractions alpha(m, x, y), precomputed at create over the same
    // per-level boxes as the force terms (frc_off / 2 = cell offset); null: no obstacle
    const double* alpha_tab;
    // near-threshold tie log (north_star): records of group metrics within
    // 1e-12 relative of eps_l or 2^{mu+d} eps_l; step_no = steps completed since commit
    mrlbm_tie_record* ties;
    int* tie_n;
    int tie_cap;
    const int* step_no;
    long long frc_off[kL];
    int frc_x0[kL], frc_y0[kL], frc_nx[kL], frc_ny[kL];
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ int mr_coord(int c, int n, int per)
{
    if (per)
    {
        c %= n;
        return c < 0 ? c + n : c;
    }
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

template <int D>
__device__ __forceinline__ void lin2xy(int lin, int ny, int& x, int& y)
{
    if (D == 1)
    {
        x = lin;
        y = 0;
    }
    else
    {
        x = lin / ny;
        y = lin - x * ny;
    }
}

// same with a shift when the row length is a power of two (all BASELINE configs)
template <int D>
__device__ __forceinline__ void lin2xy_l(int lin, int ny, int lny, int& x, int& y)
{
    if (D == 1)
    {
        x = lin;
        y = 0;
    }
    else if (lny >= 0)
    {
        x = lin >> lny;
        y = lin & (ny - 1);
    }
    else
    {
        x = lin / ny;
        y = lin - x * ny;
    }
}

template <int D>
__device__ __forceinline__ int xy2lin(int x, int y, int ny)
{
    return D == 1 ? x : x * ny + y;
}

// Value layout: the fp64 population arrays are stored in 2x2 sibling
// blocks -- the 2^D children of a cell, in children order (dx, dy) = (c >> 1, c & 1),
// are 2^D consecutive doubles (one 32-byte sector per population in 2D), blocks
// row-major over the parents.  Kinds / flags / slot lists stay row-major (lin).
template <int D>
__device__ __forceinline__ int vix(int x, int y, int ny)
{
    if (D == 1)
        return x;
    return (((x >> 1) * (ny >> 1) + (y >> 1)) << 2) + ((x & 1) << 1) + (y & 1);
}

// value index of a row-major linear index
template <int D>
__device__ __forceinline__ int vl(int lin, int ny, int lny)
{
    if (D == 1)
        return lin;
    int x, y;
    if (lny >= 0)
    {
        x = lin >> lny;
        y = lin & (ny - 1);
    }
    else
    {
        x = lin / ny;
        y = lin - x * ny;
    }
    return vix<D>(x, y, ny);
}

// the 2^D children of cell (px, py) in children order: one sibling block, read as
// 16-byte loads from one 32-byte sector (2D) / one 16-byte load (1D)
template <int D>
__device__ __forceinline__ void load_children(const double* __restrict__ src, int px, int py, int ny1,
                                              double (&ch)[1 << D])
{
    if (D == 1)
    {
        const double2 a = *reinterpret_cast<const double2*>(src + 2 * px);
        ch[0] = a.x;
        ch[1] = a.y;
    }
    else
    {
        const double* b0 = src + (((long long)px * (ny1 >> 1) + py) << 2);
        const double2 a = *reinterpret_cast<const double2*>(b0);
        const double2 b = *reinterpret_cast<const double2*>(b0 + 2);
        ch[0] = a.x;
        ch[1] = a.y;
        ch[D == 1 ? 1 : 2] = b.x;
        ch[D == 1 ? 1 : 3] = b.y;
    }
}

// stencil lookup with the MR boundary rule (clamp / wrap), Decision D.8
template <int D>
__device__ __forceinline__ int mr_lin(const Geo& g, int m, int x, int y)
{
    const int li = m - g.J0;
    const int xx = mr_coord(x, g.nx[li], g.per0);
    if (D == 1)
        return xx;
    const int yy = mr_coord(y, g.ny[li], g.per1);
    return xx * g.ny[li] + yy;
}

// same, value index
template <int D>
__device__ __forceinline__ int mr_vix(const Geo& g, int m, int x, int y)
{
    const int li = m - g.J0;
    const int xx = mr_coord(x, g.nx[li], g.per0);
    if (D == 1)
        return xx;
    const int yy = mr_coord(y, g.ny[li], g.per1);
    return vix<D>(xx, yy, g.ny[li]);
}

// reference predict<D> operation order (prediction.hpp:64-75, 143-159), gamma = 1
// st: 3 (1D) or 9 (2D, index (ox+1)*3 + (oy+1)) stencil values
template <int D>
__device__ __forceinline__ double mr_predict(const double* st, int dx, int dy)
{
    const double c1 = -0.125;
    const double center = st[D == 1 ? 1 : 4];
    if (D == 1)
    {
        const double s0 = dx == 0 ? 1.0 : -1.0;
        const double q1 = __dadd_rn(0.0, __dmul_rn(c1, __dsub_rn(st[2], st[0])));
        return __dadd_rn(center, __dmul_rn(s0, q1));
    }
    else
    {
        const double s0 = dx == 0 ? 1.0 : -1.0;
        const double s1 = dy == 0 ? 1.0 : -1.0;
        const double qx = __dadd_rn(0.0, __dmul_rn(c1, __dsub_rn(st[7], st[1])));
        const double qy = __dadd_rn(0.0, __dmul_rn(c1, __dsub_rn(st[5], st[3])));
        const double inner = __dadd_rn(__dsub_rn(__dsub_rn(st[8], st[2]), st[6]), st[0]);
        const double qxy = __dadd_rn(0.0, __dmul_rn(__dmul_rn(c1, c1), inner));
        const double a = __dadd_rn(__dadd_rn(center, __dmul_rn(s0, qx)), __dmul_rn(s1, qy));
        return __dsub_rn(a, __dmul_rn(__dmul_rn(s0, s1), qxy));
    }
}

// generated unrolled table sums for the built-in velocity sets (gen_stream.py)
#include "stream_gen.cuh"

__device__ __forceinline__ void flag_err(int* err, int which)
{
    atomicAdd(&err[which], 1);
}

// warp-aggregated append: the lanes that arrive together and target the same counter
// (same key) share one atomicAdd; lanes of one call site may append to different lists
__device__ __forceinline__ int agg_inc(int* ctr, unsigned key)
{
    const cg::coalesced_group arrived = cg::coalesced_threads();
    const cg::coalesced_group grp = cg::labeled_partition(arrived, key);
    int base = 0;
    if (grp.thread_rank() == 0)
        base = atomicAdd(ctr, (int)grp.size());
    base = grp.shfl(base, 0);
    return base + (int)grp.thread_rank();
}

// Near-threshold tie logging (BASELINE north_star: a mesh may differ from the CPU run
// only where a detail lies within 1e-12 relative of its threshold, and every such case
// is logged).  The comparison itself stays inclusive (>=,
// SPEC.md:247); this only records the group.  Same expression as the oracle's
// (oracle/mrlbm_oracle.cpp, tie_check), no FMA on either side.
__device__ __forceinline__ void tie_check(const Aux& aux, int l, int px, int py, int which, double metric, double thr)
{
    if (!(thr > 0.0) || !(fabs(__dsub_rn(metric, thr)) <= __dmul_rn(1e-12, thr)))
        return;
    const int k = atomicAdd(aux.tie_n, 1);
    if (k < aux.tie_cap)
    {
        mrlbm_tie_record r;
        r.step = *aux.step_no + 1;
        r.level = l;
        r.cell[0] = px;
        r.cell[1] = py;
        r.cell[2] = 0;
        r.which = which;
        r.metric = metric;
        r.threshold = thr;
        aux.ties[k] = r;
    }
}

#define GRID_STRIDE(i, begin, end)                                                                  \
    for (long long i = (long long)(begin) + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)(end); \
         i += (long long)gridDim.x * blockDim.x)

// Multi-level launches: one grid covers several levels; block ranges per level are
// prefix sums computed on the host.  Each block derives its level and its block
// index / count within the level (grid-stride loops then run per level).
struct LGrid {
    int start[kL + 1];
    int m0, nl;
};

__device__ __forceinline__ void lgrid_setup(const LGrid& lg, int& m, int& lvb, int& lvg)
{
    int i = 0;
    while (i + 1 < lg.nl && (int)blockIdx.x >= lg.start[i + 1])
        ++i;
    m = lg.m0 + i;
    lvb = (int)blockIdx.x - lg.start[i];
    lvg = lg.start[i + 1] - lg.start[i];
}

#define LGRID_STRIDE(i, begin, end)                                                                                  \
    for (long long i = (long long)(begin) + (long long)lvb_ * blockDim.x + threadIdx.x; i < (long long)(end);      \
         i += (long long)lvg_ * blockDim.x)
#define LSETUP                                                                                                      \
    int m, lvb_, lvg_;                                                                                              \
    lgrid_setup(lg_, m, lvb_, lvg_)

struct TileP {
    int* t[kL];
};

// zero the per-step keep / rn flags of every level (16 bytes per thread)
__global__ void k_zero_flags(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_, int* fbc)
{
    LSETUP;
    const int li = m - g.J0;
    const long long n16 = g.cap[li] / 16, n = g.cap[li];
    if (blockIdx.x == 0 && threadIdx.x < 8)
        fbc[threadIdx.x] = 0;
    LGRID_STRIDE(i, 0, n16)
    {
        reinterpret_cast<uint4*>(fl.keep[li])[i] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4*>(fl.rn[li])[i] = make_uint4(0, 0, 0, 0);
    }
    if (lvb_ == 0)
        for (long long i = n16 * 16 + threadIdx.x; i < n; i += blockDim.x)
        {
            fl.keep[li][i] = 0;
            fl.rn[li][i] = 0;
        }
}

// ---------------------------------------------------------------- K1 / K6 project
// internal value = (sum of the 2^D children in children order) / 2^D   (prediction.hpp:51-60)
template <int D, int Q>
__global__ void __launch_bounds__(256) k_project(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Fld F, int m, const __grid_constant__ Aux aux)
{
    const int li = m - g.J0;
    const int nL = t.cnt[li * 4 + 0], nI = t.cnt[li * 4 + 1];
    const int ny = g.ny[li], ny1 = g.ny[li + 1];
    const long long cap = g.cap[li], cap1 = g.cap[li + 1];
    GRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = t.cells[li][s];
        int px, py;
        lin2xy_l<D>(plin, ny, g.lny[li], px, py);
        int cs[1 << D];
        for (int c = 0; c < (1 << D); ++c)
        {
            const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
            cs[c] = xy2lin<D>(2 * px + dx, 2 * py + dy, ny1);
        }
        double v[Q];
#pragma unroll
        for (int h = 0; h < Q; ++h)
        {
            double ch[1 << D];
            load_children<D>(F.f[li + 1] + (long long)h * cap1, px, py, ny1, ch);
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < (1 << D); ++c)
                acc = __dadd_rn(acc, ch[c]);
            v[h] = __ddiv_rn(acc, (double)(1 << D));
        }
        const int pv = vix<D>(px, py, ny);
#pragma unroll
        for (int h = 0; h < Q; ++h)
            F.f[li][(long long)h * cap + pv] = v[h];
    }
}

// K6: projection of the new tree, restricted to "dirty" internal nodes.  A node is
// dirty if it is new to the complete tree or one of its children is dirty; a clean
// node keeps the value K1 computed this step (same children, same values, same
// summation order -> bit-identical).  dirty[] (per level, written for every new
// internal node) carries the flag bottom-up; leaves are dirty iff not in the old tree.
template <int D, int Q>
__global__ void __launch_bounds__(256) k_project_new(const __grid_constant__ Geo g, const __grid_constant__ Tree to, const __grid_constant__ Tree tn, const __grid_constant__ Fld F, int m, uint8_t* const* dirty)
{
    const int li = m - g.J0;
    const int nL = tn.cnt[li * 4 + 0], nI = tn.cnt[li * 4 + 1];
    const int ny = g.ny[li], ny1 = g.ny[li + 1];
    const long long cap = g.cap[li], cap1 = g.cap[li + 1];
    const uint8_t* dchild = dirty[li + 1];
    GRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = tn.cells[li][s];
        int px, py;
        lin2xy_l<D>(plin, ny, g.lny[li], px, py);
        int cs[1 << D];
        bool d = !(to.kind[li][plin] & (K_LEAF | K_INT));
        for (int c = 0; c < (1 << D); ++c)
        {
            const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
            cs[c] = xy2lin<D>(2 * px + dx, 2 * py + dy, ny1);
            const uint8_t kc = tn.kind[li + 1][cs[c]];
            d = d || ((kc & K_INT) ? dchild[cs[c]] != 0 : !(to.kind[li + 1][cs[c]] & (K_LEAF | K_INT)));
        }
        dirty[li][plin] = d;
        if (!d)
            continue;
        double v[Q];
#pragma unroll
        for (int h = 0; h < Q; ++h)
        {
            double ch[1 << D];
            load_children<D>(F.f[li + 1] + (long long)h * cap1, px, py, ny1, ch);
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < (1 << D); ++c)
                acc = __dadd_rn(acc, ch[c]);
            v[h] = __ddiv_rn(acc, (double)(1 << D));
        }
        const int pv = vix<D>(px, py, ny);
#pragma unroll
        for (int h = 0; h < Q; ++h)
            F.f[li][(long long)h * cap + pv] = v[h];
    }
}

// ---------------------------------------------------------------- K2 details
// d = f - predict; metric = max over siblings and populations
// (PAPER.md:656); keep iff metric >= eps_l (Eq. 10), blow-up
// refinement iff metric >= 2^{mu+D} eps_l
template <int D, int Q>
__global__ void __launch_bounds__(256, 4) k_details(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Fld F, const __grid_constant__ Flags fl, const SchemeDev* sc, const __grid_constant__ LGrid lg_, const __grid_constant__ Aux aux)
{
    LSETUP;
    const int li = m - g.J0;
    const int l = m + 1;
    const int nL = t.cnt[li * 4 + 0], nI = t.cnt[li * 4 + 1];
    const int ny = g.ny[li], ny1 = g.ny[li + 1];
    const long long cap = g.cap[li], cap1 = g.cap[li + 1];
    const double eps_l = ldexp(sc->eps, D * (l - g.J1));
    const double eps_b = ldexp(eps_l, sc->mu + D);
    const bool can_b = (l > g.J0) && (l < g.J1);
    LGRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = t.cells[li][s];
        int px, py;
        lin2xy_l<D>(plin, ny, g.lny[li], px, py);
        constexpr int NS = D == 1 ? 3 : 9;
        int st[NS];
        bool ok = true;
        for (int o = 0; o < NS; ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            const int lin = mr_lin<D>(g, m, px + ox, py + oy);
            st[o] = mr_vix<D>(g, m, px + ox, py + oy);
            ok = ok && (t.kind[li][lin] & (K_LEAF | K_INT)); // grading: the stencil is in R
        }
        int cs[1 << D];
        for (int c = 0; c < (1 << D); ++c)
        {
            const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
            cs[c] = xy2lin<D>(2 * px + dx, 2 * py + dy, ny1);
        }
        if (!ok)
        {
            flag_err(aux.err, 0);
            continue;
        }
        double metric = 0.0;
        #pragma unroll 3
        for (int h = 0; h < Q; ++h)
        {
            const double* fm = F.f[li] + (long long)h * cap;
            const double* f1 = F.f[li + 1] + (long long)h * cap1;
            double sv[NS];
            for (int o = 0; o < NS; ++o)
                sv[o] = fm[st[o]];
            double ch[1 << D];
            load_children<D>(f1, px, py, ny1, ch);
#pragma unroll
            for (int c = 0; c < (1 << D); ++c)
            {
                const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
                const double d = __dsub_rn(ch[c], mr_predict<D>(sv, dx, dy));
                const double ad = fabs(d);
                if (ad > metric)
                    metric = ad;
            }
        }
        tie_check(aux, l, px, py, 0, metric, eps_l);
        if (can_b)
            tie_check(aux, l, px, py, 1, metric, eps_b);
        if (metric >= eps_l)
            fl.keep[li][plin] = 1;
        if (can_b && metric >= eps_b)
        {
            // H(b): refine the 2^D children of every cell of the group
            for (int c = 0; c < (1 << D); ++c)
            {
                const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
                fl.rn[li + 1][xy2lin<D>(2 * px + dx, 2 * py + dy, ny1)] = 1;
            }
        }
    }
}

// K1+K2 fused, one launch per level (m = J1-1 .. J0, bottom-up): each internal node
// p of the old tree at level m projects its children (written: K6, the transfer and
// the next level need it) and computes the details of its sibling group against the
// prediction from its 3^D stencil at level m.  Internal stencil neighbours are
// projected again in registers from their own children -- the same sum in children
// order and division as their own thread, so bit-identical -- instead of reading the
// value back after a grid-wide barrier: the children blocks are read once from DRAM
// (neighbours' blocks are adjacent sectors, L1/L2 hits).
template <int D>
__device__ __forceinline__ double proj_block(const double* __restrict__ src, int base)
{
    double acc = 0.0;
    if (D == 1)
    {
        const double2 a = *reinterpret_cast<const double2*>(src + base);
        acc = __dadd_rn(__dadd_rn(acc, a.x), a.y);
    }
    else
    {
        const double2 a = *reinterpret_cast<const double2*>(src + base);
        const double2 b = *reinterpret_cast<const double2*>(src + base + 2);
        acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, a.x), a.y), b.x), b.y);
    }
    return __ddiv_rn(acc, (double)(1 << D));
}

template <int D, int Q>
__global__ void __launch_bounds__(256, 3)
    k_proj_details(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Fld F,
                   const __grid_constant__ Flags fl, const SchemeDev* sc, int m, const __grid_constant__ Aux aux)
{
    const int li = m - g.J0;
    const int l = m + 1;
    const int nL = t.cnt[li * 4 + 0], nI = t.cnt[li * 4 + 1];
    const int nx = g.nx[li], ny = g.ny[li], ny1 = g.ny[li + 1];
    const long long cap = g.cap[li], cap1 = g.cap[li + 1];
    const double eps_l = ldexp(sc->eps, D * (l - g.J1));
    const double eps_b = ldexp(eps_l, sc->mu + D);
    const bool can_b = (l > g.J0) && (l < g.J1);
    constexpr int NS = D == 1 ? 3 : 9;
    constexpr int C = D == 1 ? 1 : 4; // stencil centre
    GRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = t.cells[li][s];
        int px, py;
        lin2xy_l<D>(plin, ny, g.lny[li], px, py);
        // stencil sources: value index at level m (leaf) or -1 - child block (internal)
        int src[NS];
        bool ok = true;
        for (int o = 0; o < NS; ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            const int xx = mr_coord(px + ox, nx, g.per0);
            const int yy = D == 1 ? 0 : mr_coord(py + oy, ny, g.per1);
            const uint8_t kd = t.kind[li][xy2lin<D>(xx, yy, ny)];
            ok = ok && (kd & (K_LEAF | K_INT)); // grading: the stencil is in R
            src[o] = (kd & K_INT) ? -1 - (D == 1 ? 2 * xx : ((xx * (ny1 >> 1) + yy) << 2)) : vix<D>(xx, yy, ny);
        }
        const int pv = vix<D>(px, py, ny);
        const int cb = D == 1 ? 2 * px : ((px * (ny1 >> 1) + py) << 2);
        double metric = 0.0;
#pragma unroll 1
        for (int h = 0; h < Q; ++h)
        {
            const double* fm = F.f[li] + (long long)h * cap;
            const double* f1 = F.f[li + 1] + (long long)h * cap1;
            double ch[1 << D];
            load_children<D>(f1, px, py, ny1, ch);
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < (1 << D); ++c)
                acc = __dadd_rn(acc, ch[c]);
            const double centre = __ddiv_rn(acc, (double)(1 << D));
            F.f[li][(long long)h * cap + pv] = centre;
            double sv[NS];
#pragma unroll
            for (int o = 0; o < NS; ++o)
            {
                if (o == C)
                    sv[o] = centre;
                else
                    sv[o] = src[o] >= 0 ? fm[src[o]] : proj_block<D>(f1, -1 - src[o]);
            }
            (void)cb;
#pragma unroll
            for (int c = 0; c < (1 << D); ++c)
            {
                const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
                const double d = __dsub_rn(ch[c], mr_predict<D>(sv, dx, dy));
                const double ad = fabs(d);
                if (ad > metric)
                    metric = ad;
            }
        }
        if (!ok)
        {
            flag_err(aux.err, 0);
            continue;
        }
        tie_check(aux, l, px, py, 0, metric, eps_l);
        if (can_b)
            tie_check(aux, l, px, py, 1, metric, eps_b);
        if (metric >= eps_l)
            fl.keep[li][plin] = 1;
        if (can_b && metric >= eps_b)
        {
            for (int c = 0; c < (1 << D); ++c)
            {
                const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
                fl.rn[li + 1][xy2lin<D>(2 * px + dx, 2 * py + dy, ny1)] = 1;
            }
        }
    }
}

// ---------------------------------------------------------------- K3 flags
// T closure: ancestors of kept groups are kept (Decision D.4)
template <int D>
__global__ void k_closure(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Flags fl, int m)
{
    const int li = m - g.J0;
    const int nL = t.cnt[li * 4 + 0], nI = t.cnt[li * 4 + 1];
    const int ny = g.ny[li], nyp = g.ny[li - 1];
    GRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = t.cells[li][s];
        if (!fl.keep[li][plin])
            continue;
        int px, py;
        lin2xy_l<D>(plin, ny, g.lny[li], px, py);
        fl.keep[li - 1][xy2lin<D>(px >> 1, py >> 1, nyp)] = 1;
    }
}

// rn |= keep;  H(a): (l, k - eta^h) for k in R(T) at level l = m + 1
template <int D>
__global__ void k_enlarge(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Flags fl, const SchemeDev* sc, const __grid_constant__ LGrid lg_, unsigned emask)
{
    LSETUP;
    (void)sc;
    const int li = m - g.J0;
    const int nL = t.cnt[li * 4 + 0], nI = t.cnt[li * 4 + 1];
    const int ny = g.ny[li];
    LGRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = t.cells[li][s];
        if (!fl.keep[li][plin])
            continue;
        fl.rn[li][plin] = 1;
        int px, py;
        lin2xy_l<D>(plin, ny, g.lny[li], px, py);
        // distinct parents of the shifted children: a static 3^D offset mask (emask);
        // a target parent inside the domain always has an in-domain contributing child
        const int nx = g.nx[li];
        for (int o = 0; o < 9; ++o)
        {
            if (!((emask >> o) & 1u))
                continue;
            const int ox = o / 3 - 1, oy = o % 3 - 1;
            int x = px + ox, y = py + (D == 1 ? 0 : oy);
            if (!g.per0 && (x < 0 || x >= nx))
                continue;
            if (D == 2 && !g.per1 && (y < 0 || y >= ny))
                continue;
            x = mr_coord(x, nx, 1);
            if (D == 2)
                y = mr_coord(y, ny, 1);
            fl.rn[li][xy2lin<D>(x, y, ny)] = 1;
        }
    }
}

union V16 {
    uint4 v;
    uint8_t b[16];
};

// T closure as a gather (2D, 16 parents of a row per thread): keep(p) |= OR of the
// keep flags of p's 2x2 children at level m (keep is only ever set on internal nodes)
__global__ void k_closure_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, int m)
{
    const int li = m - g.J0; // children level
    const int nyp = g.ny[li - 1], ny = g.ny[li];
    const long long nch = (long long)g.nx[li - 1] * nyp / 16;
    const uint8_t* kc = fl.keep[li];
    uint8_t* kp = fl.keep[li - 1];
    GRID_STRIDE(c, 0, nch)
    {
        const int lin0 = (int)(c * 16);
        const int px = lin0 >> g.lny[li - 1], py0 = lin0 & (nyp - 1);
        const uint4* r0 = reinterpret_cast<const uint4*>(kc + (long long)(2 * px) * ny + 2 * py0);
        const uint4* r1 = reinterpret_cast<const uint4*>(kc + (long long)(2 * px + 1) * ny + 2 * py0);
        V16 a0, a1, b0, b1;
        a0.v = r0[0];
        a1.v = r0[1];
        b0.v = r1[0];
        b1.v = r1[1];
        if (((a0.v.x | a0.v.y | a0.v.z | a0.v.w) | (a1.v.x | a1.v.y | a1.v.z | a1.v.w) |
             (b0.v.x | b0.v.y | b0.v.z | b0.v.w) | (b1.v.x | b1.v.y | b1.v.z | b1.v.w)) == 0)
            continue;
        V16 o;
#pragma unroll
        for (int j = 0; j < 16; ++j)
        {
            const V16& A = j < 8 ? a0 : a1;
            const V16& B = j < 8 ? b0 : b1;
            const int k = 2 * (j & 7);
            o.b[j] = A.b[k] | A.b[k + 1] | B.b[k] | B.b[k + 1];
        }
        uint4* dst = reinterpret_cast<uint4*>(kp) + c;
        const uint4 cur = *dst;
        *dst = make_uint4(cur.x | o.v.x, cur.y | o.v.y, cur.z | o.v.z, cur.w | o.v.w);
    }
}

// same as a gather over a dense level (2D, 16 cells of a row per thread): rn(c) |=
// keep(c) | OR over the emask offsets o of keep(c - o), wrap on periodic axes, nothing
// from outside the domain otherwise -- the set k_enlarge scatters, without per-parent
// scattered byte stores
__global__ void k_enlarge_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl,
                            const __grid_constant__ LGrid lg_, unsigned emask)
{
    LSETUP;
    const int li = m - g.J0;
    const int nx = g.nx[li], ny = g.ny[li];
    const long long nch = (long long)nx * ny / 16;
    const uint8_t* keep = fl.keep[li];
    uint8_t* rn = fl.rn[li];
    LGRID_STRIDE(c, 0, nch)
    {
        const int lin0 = (int)(c * 16);
        const int x = lin0 >> g.lny[li], y0 = lin0 & (ny - 1);
        // keep of rows x-1, x, x+1 over columns y0-1 .. y0+16
        uint8_t w[3][18];
        bool any = false;
#pragma unroll
        for (int r = 0; r < 3; ++r)
        {
            int xr = x + r - 1;
            const bool ok = (xr >= 0 && xr < nx) || g.per0;
            xr = mr_coord(xr, nx, 1);
            V16 v;
            v.v = ok ? reinterpret_cast<const uint4*>(keep + (long long)xr * ny)[y0 >> 4] : make_uint4(0, 0, 0, 0);
            any = any || (v.v.x | v.v.y | v.v.z | v.v.w);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                w[r][j + 1] = v.b[j];
            const int yl = y0 - 1, yr = y0 + 16;
            w[r][0] = (ok && (yl >= 0 || g.per1)) ? keep[(long long)xr * ny + mr_coord(yl, ny, 1)] : 0;
            w[r][17] = (ok && (yr < ny || g.per1)) ? keep[(long long)xr * ny + mr_coord(yr, ny, 1)] : 0;
            any = any || w[r][0] || w[r][17];
        }
        if (!any)
            continue;
        V16 o;
#pragma unroll
        for (int j = 0; j < 16; ++j)
        {
            uint8_t v = w[1][j + 1];
#pragma unroll
            for (int b = 0; b < 9; ++b)
                if ((emask >> b) & 1u)
                {
                    const int ox = b / 3 - 1, oy = b % 3 - 1;
                    v |= w[1 - ox][j + 1 - oy];
                }
            o.b[j] = v;
        }
        uint4* dst = reinterpret_cast<uint4*>(rn) + c;
        const uint4 cur = *dst;
        *dst = make_uint4(cur.x | o.v.x, cur.y | o.v.y, cur.z | o.v.z, cur.w | o.v.w);
    }
}

// grading G: for p refined at level m, its 3^D box must be in R_m, i.e. the
// parents of the box at level m-1 are refined (one fine->coarse sweep, Decision D.7)
template <int D>
__global__ void k_grade(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, int m)
{
    const int li = m - g.J0;
    const int nx = g.nx[li], ny = g.ny[li], nyp = g.ny[li - 1];
    const long long n = (long long)nx * ny;
    GRID_STRIDE(i, 0, n)
    {
        if (!fl.rn[li][i])
            continue;
        int px, py;
        lin2xy_l<D>((int)i, ny, g.lny[li], px, py);
        // the parents of the 3^D box: the distinct values of (px +- 1) >> 1 per axis
        // (px >> 1 is always one of them; an out-of-domain neighbour adds nothing)
        auto par = [](int c, int o, int n, int per) {
            int v = c + o;
            if (v < 0 || v >= n)
            {
                if (!per)
                    return c >> 1;
                v = mr_coord(v, n, 1);
            }
            return v >> 1;
        };
        const int ax0 = par(px, -1, nx, g.per0), ax1 = par(px, 1, nx, g.per0);
        const int ay0 = D == 2 ? par(py, -1, ny, g.per1) : 0, ay1 = D == 2 ? par(py, 1, ny, g.per1) : 0;
        for (int a = 0; a < (ax1 != ax0 ? 2 : 1); ++a)
            for (int b = 0; b < (ay1 != ay0 ? 2 : 1); ++b)
                fl.rn[li - 1][xy2lin<D>(a ? ax1 : ax0, b ? ay1 : ay0, nyp)] = 1;
    }
}

// same, 16 cells of a row per thread (one 16-byte load; empty chunks cost one load)
__global__ void k_grade_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, int m)
{
    const int li = m - g.J0;
    const int nx = g.nx[li], ny = g.ny[li], nyp = g.ny[li - 1];
    const long long nch = (long long)nx * ny / 16;
    const uint8_t* rn = fl.rn[li];
    uint8_t* rnp = fl.rn[li - 1];
    GRID_STRIDE(c, 0, nch)
    {
        const uint4 v = reinterpret_cast<const uint4*>(rn)[c];
        if ((v.x | v.y | v.z | v.w) == 0)
            continue;
        const int lin0 = (int)(c * 16);
        const int px = lin0 >> g.lny[li], y0 = lin0 & (ny - 1);
        // distinct parent rows of px-1..px+1 (clipped / wrapped)
        int prow[3], npr = 0;
        for (int o = -1; o <= 1; ++o)
        {
            int xv = px + o;
            if (xv < 0 || xv >= nx)
            {
                if (!g.per0)
                    continue;
                xv = mr_coord(xv, nx, 1);
            }
            const int r = xv >> 1;
            bool dup = false;
            for (int k = 0; k < npr; ++k)
                dup = dup || prow[k] == r;
            if (!dup)
                prow[npr++] = r;
        }
        // parent columns touched by the set cells' y-1..y+1: a bit mask over
        // (y0 - 1) >> 1 .. (y0 + 16) >> 1 plus wrapped ends
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
        unsigned cols = 0; // bit j: parent column (y0 >> 1) - 1 + j, j in [0, 10)
        bool wrapLo = false, wrapHi = false;
        for (int j = 0; j < 16; ++j)
        {
            if (!b[j])
                continue;
            const int y = y0 + j;
            for (int o = -1; o <= 1; ++o)
            {
                const int yv = y + o;
                if (yv < 0)
                {
                    if (g.per1)
                        wrapLo = true;
                    continue;
                }
                if (yv >= ny)
                {
                    if (g.per1)
                        wrapHi = true;
                    continue;
                }
                cols |= 1u << ((yv >> 1) - (y0 >> 1) + 1);
            }
        }
        for (int k = 0; k < npr; ++k)
        {
            uint8_t* row = rnp + (long long)prow[k] * nyp;
            for (int j = 0; j < 10; ++j)
                if ((cols >> j) & 1u)
                    row[(y0 >> 1) - 1 + j] = 1;
            if (wrapLo)
                row[mr_coord(-1, ny, 1) >> 1] = 1;
            if (wrapHi)
                row[mr_coord(ny, ny, 1) >> 1] = 1;
        }
    }
}

// The deep-gap (gap >= 2) fallback leaves of levels J0..J1-2, listed tile by tile
// (16 x 16 cells, tile order inside, one atomicAdd per tile) with their table masks:
// K8 gives each warp 32 consecutive list entries for one population, so the warp's
// leaves are spatial neighbours and their box / rim loads share sectors.  (Appended
// from the classification kernel in arrival order, K8 read 3.0 GB of DRAM per
// transient step at an L2 hit rate of 19 %.)  Multi-level launch; the order of the
// tiles in the list is unspecified and no result depends on it.
constexpr int kLongGap = 4; // K8: gap from which a leaf's rims are evaluated by a whole warp
// The warp-cooperative launch wins when the long-rim leaves are few (their serial chains
// set the duration of the thread kernel: settled regime 404 -> 150 us, transient window
// 1089 -> 872 us) and loses when they are many (developing flow, thousands of gap-4 / 5
// leaves: 331 -> 436 us serialised), so the threshold moves up by kLongStep levels when more
// than kLongMany leaves lie at or above it.  (With the two launches on forked streams a
// step of 1 -- gap >= 5 in the warp launch, 229 us, beside gap 2..4 in the thread launch,
// 168 us -- still lost to a step of 2 at step 3000: 1.345 vs 1.297 ms per step.)  Counted
// per step by k_list_deep (fb_count[5]: gap >= k8_long, fb_count[6]: gap >= k8_long +
// kLongStep); both K8 launches evaluate the same rule.
constexpr int kLongMany = 2048;
constexpr int kLongStep = 2;
__device__ __forceinline__ int k8_long_gap(int base, const int* fb_count)
{
    return (base > 0 && fb_count[5] > kLongMany) ? base + kLongStep : base;
}

template <int D>
__global__ void __launch_bounds__(256) k_list_deep(const __grid_constant__ Geo g, const __grid_constant__ Flags fl,
                                                   const __grid_constant__ LGrid lg_, const __grid_constant__ Aux aux)
{
    LSETUP;
    const int li = m - g.J0;
    const int nx = g.nx[li], ny = D == 1 ? 1 : g.ny[li];
    const int tny = D == 1 ? 1 : (ny + 15) >> 4;
    const long long ntiles = D == 1 ? ((long long)nx + 255) / 256 : (long long)((nx + 15) >> 4) * tny;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int woff[8];
    __shared__ int sbase, slong;
    const bool longrim = aux.k8_long > 0 && g.J1 - m >= aux.k8_long;
    for (long long t = lvb_; t < ntiles; t += lvg_)
    {
        int x, y;
        if (D == 1)
        {
            x = (int)t * 256 + threadIdx.x;
            y = 0;
        }
        else
        {
            const int tx = (int)(t / tny), ty = (int)(t - (long long)tx * tny);
            x = tx * 16 + (threadIdx.x >> 4);
            y = ty * 16 + (threadIdx.x & 15);
        }
        bool pick = false;
        int lin = 0;
        if (x < nx && y < ny)
        {
            lin = xy2lin<D>(x, y, ny);
            pick = fl.kind[li][lin] == (K_LEAF | K_FB);
        }
        const unsigned b = __ballot_sync(0xffffffffu, pick);
        if (lane == 0)
            woff[wid] = __popc(b);
        __syncthreads();
        if (threadIdx.x == 0)
        {
            int tot = 0;
            for (int w = 0; w < 8; ++w)
            {
                const int c = woff[w];
                woff[w] = tot;
                tot += c;
            }
            sbase = tot ? atomicAdd(aux.fb_count, tot) : 0;
            slong = tot && longrim ? atomicAdd(aux.fb_count + 5, tot) : 0;
            if (tot && longrim && g.J1 - m >= aux.k8_long + kLongStep)
                atomicAdd(aux.fb_count + 6, tot);
        }
        __syncthreads();
        if (pick)
        {
            const int r = woff[wid] + __popc(b & ((1u << lane) - 1u));
            const int k = sbase + r;
            // the long-rim entries (gap >= kLongGap) are also indexed from the tail of the
            // list buffer, for the warp-cooperative K8 launch; capacity = all cells, so the
            // head (<= leaves of the levels <= J1-2) and the tail never meet
            if (k < aux.fb_cap && (!longrim || (long long)k < aux.fb_cap - 1 - (slong + r)))
            {
                const int vi = vix<D>(x, y, ny);
                aux.fb_list[k] = make_int2(m, lin);
                aux.fb_mask[k] = fl.fbm[li][vi];
                aux.fb_dmask[k] = fl.fbd[li][vi];
                if (longrim)
                    aux.fb_list[aux.fb_cap - 1 - (slong + r)] = make_int2(k, m);
            }
            else
                flag_err(aux.err, 2);
        }
        __syncthreads();
    }
}

// The gap-1 fallback leaves without domain-leaving pairs (the bulk of the fallback
// leaves, K7 MODE 2), listed tile by tile: one block per 16 x 16 tile of level J1-1
// (1D: 256 cells), the tile's leaves in tile order, one atomicAdd per tile.  MODE 2
// takes consecutive list entries, so a warp's leaves are spatial neighbours and their
// 5 x 5 boxes and finest rings are L1 / L2 hits instead of DRAM re-reads.  (An append
// from the classification kernel lists them in arrival order: measured 5.9 GB of DRAM
// reads per transient step for MODE 2, L2 hit rate 19 %.)  The tiles' order in the
// list is unspecified; every leaf's result is independent of it (bit-exact).
template <int D>
__global__ void __launch_bounds__(256) k_list_fb1(const __grid_constant__ Geo g, const __grid_constant__ Flags fl,
                                                  const __grid_constant__ Aux aux)
{
    const int li = g.nlev - 2;
    const int nx = g.nx[li], ny = D == 1 ? 1 : g.ny[li];
    const int tny = D == 1 ? 1 : (ny + 15) >> 4;
    const long long ntiles = D == 1 ? ((long long)nx + 255) / 256 : (long long)((nx + 15) >> 4) * tny;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int woff[8];
    __shared__ int sbase;
    int* out = aux.fbs + aux.fbs_off[2];
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x)
    {
        int x, y;
        if (D == 1)
        {
            x = (int)t * 256 + threadIdx.x;
            y = 0;
        }
        else
        {
            const int tx = (int)(t / tny), ty = (int)(t - (long long)tx * tny);
            x = tx * 16 + (threadIdx.x >> 4);
            y = ty * 16 + (threadIdx.x & 15);
        }
        bool pick = false;
        int lin = 0;
        if (x < nx && y < ny)
        {
            lin = xy2lin<D>(x, y, ny);
            pick = fl.kind[li][lin] == (K_LEAF | K_FB) && fl.fbd[li][vix<D>(x, y, ny)] == 0u;
        }
        const unsigned b = __ballot_sync(0xffffffffu, pick);
        if (lane == 0)
            woff[wid] = __popc(b);
        __syncthreads();
        if (threadIdx.x == 0)
        {
            int tot = 0;
            for (int w = 0; w < 8; ++w)
            {
                const int c = woff[w];
                woff[w] = tot;
                tot += c;
            }
            sbase = tot ? atomicAdd(aux.fb_count + 4, tot) : 0;
        }
        __syncthreads();
        if (pick)
        {
            const int k = sbase + woff[wid] + __popc(b & ((1u << lane) - 1u));
            if (k < aux.fbs_cap[2])
                out[k] = lin;
            else
                flag_err(aux.err, 2);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- K4 kinds, fallback, ghosts, compaction
template <int D>
__global__ void k_kinds(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    const int li = m - g.J0;
    const int ny = g.ny[li], nyp = li > 0 ? g.ny[li - 1] : 1;
    const long long n = (long long)g.nx[li] * ny;
    LGRID_STRIDE(i, 0, n)
    {
        int x, y;
        lin2xy_l<D>((int)i, ny, g.lny[li], x, y);
        const bool inR = (m == g.J0) || fl.rn[li - 1][xy2lin<D>(x >> 1, y >> 1, nyp)];
        const bool ref = (m < g.J1) && fl.rn[li][i];
        fl.kind[li][i] = inR ? (ref ? K_INT : K_LEAF) : 0;
    }
}

// Table exactness (Decision D.13), per (population, side): the level-l cells the
// zero-detail recursion touches lie in the domain (or periodic) and the parents of
// the level-(l+1) cells it touches are not internal.  A leaf is a fallback leaf if
// any pair fails: tested here on the union over pairs (equivalent for "any").
// Mark the reconstruction band of every fallback leaf at every finer level as
// virtual (materialised zero-detail reconstruction): a ring of width W on both
// sides of the leaf boundary, W = 2 below the finest level (stencils of the
// level above) and W = 1 at the finest level (the E/A rims themselves).
// One warp per fallback leaf.
template <int D>
__device__ __forceinline__ int band_count(int side, int W)
{
    const int S = side + 2 * W;
    if (D == 1)
        return side <= 2 * W ? S : 4 * W;
    return side <= 2 * W ? S * S : S * S - (side - 2 * W) * (side - 2 * W);
}

template <int D>
__device__ __forceinline__ void band_cell(int t, int side, int W, int bx0, int by0, int& x, int& y)
{
    const int S = side + 2 * W;
    y = 0;
    if (D == 1)
    {
        if (side <= 2 * W)
            x = bx0 - W + t;
        else
            x = t < 2 * W ? bx0 - W + t : bx0 + side - W + (int)(t - 2 * W);
        return;
    }
    if (side <= 2 * W)
    {
        x = bx0 - W + (t / S);
        y = by0 - W + (t % S);
        return;
    }
    const int top = 2 * W * S;
    const int mid = (side - 2 * W) * 4 * W;
    if (t < top)
    {
        x = bx0 - W + (t / S);
        y = by0 - W + (t % S);
    }
    else if (t < top + mid)
    {
        const int u = t - top;
        x = bx0 + W + (u / (4 * W));
        const int c = (u % (4 * W));
        y = c < 2 * W ? by0 - W + c : by0 + side - W + (c - 2 * W);
    }
    else
    {
        const int u = t - top - mid;
        x = bx0 + side - W + (u / S);
        y = by0 - W + (u % S);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_band(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ Aux aux)
{
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int nfb = min(*aux.fb_count, (int)aux.fb_cap);
    for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nfb; it += warps)
    {
        const int2 e = aux.fb_list[it];
        const int l = e.x;
        if (l == g.J1)
            continue;
        int kx, ky;
        lin2xy_l<D>(e.y, g.ny[l - g.J0], g.lny[l - g.J0], kx, ky);
        if (l == g.J1 - 1)
            continue; // gap 1: rim values are predicted on the fly from level J1-1 (rim_value)
        // levels l+1 .. J1-1 only: the finest-level rim cells themselves are predicted on
        // the fly from this level-(J1-1) band by K8 (rim_value), the same operands and order
        // as k_virtual would use; materialising them cost a 6 M-cell finest band per
        // transient step (k_virtual, compaction) for values read once
        for (int m = l + 1; m < g.J1; ++m)
        {
            const int li = m - g.J0;
            const int nx = g.nx[li], ny = g.ny[li];
            const int side = 1 << (m - l);
            const int W = m == g.J1 ? 1 : 2;
            const int total = band_count<D>(side, W); // < 2^31: side <= 2^(J1 - J0)
            for (int t = lane; t < total; t += 32)
            {
                int x, y;
                band_cell<D>(t, side, W, kx * side, ky * side, x, y);
                if (!g.per0 && (x < 0 || x >= nx))
                    continue;
                if (D == 2 && !g.per1 && (y < 0 || y >= ny))
                    continue;
                x = mr_coord(x, nx, 1);
                if (D == 2)
                    y = mr_coord(y, ny, 1);
                const int lin = xy2lin<D>(x, y, ny);
                if ((fl.kind[li][lin] & (K_LEAF | K_INT)) == 0)
                    fl.kind[li][lin] = K_VIRT;
            }
        }
    }
}

// ghost layer: cells not in R within Chebyshev distance gd of an R cell, gd = 2 below
// the finest level (the 5^d table boxes and the predictions of the next level's ghosts
// reach that far), gd = 1 at the finest level (only the gap-0 stream reads its ghosts:
// the 3^d neighbours; any other finest-level value is predicted on the fly, rim_value).
// 2D: separable dilation, pass 1 ORs R-membership over y +-gd into tmp, pass 2
// ORs tmp over x +-gd (10 byte reads per cell instead of 25).
__device__ __forceinline__ int ghost_dist(const Geo& g, int m)
{
    return m == g.J1 ? 1 : 2;
}

template <int D>
__global__ void k_ghost_rows(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    const int li = m - g.J0;
    uint8_t* tmp = fl.keep[li];
    const int nx = g.nx[li], ny = g.ny[li];
    const long long n = (long long)nx * ny;
    LGRID_STRIDE(i, 0, n)
    {
        int x, y;
        lin2xy_l<D>((int)i, ny, g.lny[li], x, y);
        uint8_t r = 0;
        const int gd = ghost_dist(g, m);
#pragma unroll
        for (int oy = -2; oy <= 2; ++oy)
        {
            if (oy < -gd || oy > gd)
                continue;
            int yy = y + oy;
            if (yy < 0 || yy >= ny)
            {
                if (!g.per1)
                    continue;
                yy = mr_coord(yy, ny, 1);
            }
            r |= fl.kind[li][xy2lin<D>(x, yy, ny)];
        }
        tmp[i] = r & (K_LEAF | K_INT);
    }
}

template <int D>
__global__ void k_ghost(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    const int li = m - g.J0;
    const uint8_t* tmp = fl.keep[li];
    const int nx = g.nx[li], ny = g.ny[li];
    const long long n = (long long)nx * ny;
    LGRID_STRIDE(i, 0, n)
    {
        if (fl.kind[li][i] != 0)
            continue;
        int x, y;
        lin2xy_l<D>((int)i, ny, g.lny[li], x, y);
        bool near = false;
        const int gd = ghost_dist(g, m);
#pragma unroll
        for (int ox = -2; ox <= 2; ++ox)
        {
            if (ox < -gd || ox > gd)
                continue;
            int xx = x + ox;
            if (xx < 0 || xx >= nx)
            {
                if (!g.per0)
                    continue;
                xx = mr_coord(xx, nx, 1);
            }
            if (D == 2)
                near = near || tmp[xy2lin<D>(xx, y, ny)] != 0;
            else
                near = near || (fl.kind[li][xx] & (K_LEAF | K_INT)) != 0;
        }
        if (near)
            fl.kind[li][i] = K_VIRT;
    }
}

// ---- vectorised dense passes (2D levels with ny % 16 == 0): 16 cells per thread
// per iteration with 16-byte loads, so sparse levels cost one load per 16 cells.
// Same results as the scalar kernels above.
#define CHUNK_STRIDE(c, nchunks)                                                                            \
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < (nchunks);                    \
         c += (long long)gridDim.x * blockDim.x)


__global__ void k_kinds_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    const int li = m - g.J0;
    const int ny = g.ny[li], nyp = li > 0 ? g.ny[li - 1] : 1;
    const long long nch = (long long)g.nx[li] * ny / 16;
    const uint8_t* rn = fl.rn[li];
    const uint8_t* rnp = li > 0 ? fl.rn[li - 1] : nullptr;
    const bool top = m == g.J0, fin = m == g.J1;
    LGRID_STRIDE(c, 0, nch)
    {
        const int lin0 = (int)(c * 16);
        const int x = lin0 >> g.lny[li], y0 = lin0 & (ny - 1);
        V16 r, o;
        r.v = fin ? make_uint4(0, 0, 0, 0) : reinterpret_cast<const uint4*>(rn)[c];
        uint2 pr = make_uint2(0, 0);
        if (!top)
            pr = *reinterpret_cast<const uint2*>(rnp + (long long)(x >> 1) * nyp + (y0 >> 1));
        const uint8_t* pb = reinterpret_cast<const uint8_t*>(&pr);
#pragma unroll
        for (int j = 0; j < 16; ++j)
        {
            const bool inR = top || pb[j >> 1];
            o.b[j] = inR ? (r.b[j] ? K_INT : K_LEAF) : 0;
        }
        reinterpret_cast<uint4*>(fl.kind[li])[c] = o.v;
    }
}

// fallback flags: chunks without a plain leaf are skipped with one load
template <int D>
__device__ __forceinline__ void fallback_cell(const Geo& g, const Flags& fl, int m, int li, int gap, long long i, int x,
                                              int y, const int4& ub, const int2& pi, const Aux& aux, int ib_in = -1,
                                              const int4* sdep = nullptr, const unsigned short* spm = nullptr)
{
    (void)pi;
    const int nx = g.nx[li], ny = g.ny[li];
    // internal cells of the 3^d box as bits (outside a non-periodic wall: not internal,
    // the domain test covers those)
    unsigned ib = ib_in >= 0 ? (unsigned)ib_in : 0u;
    const unsigned um = aux.umask[gap];
    if (um && ib_in < 0)
        for (int o = 0; o < (D == 1 ? 3 : 9); ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            const int bit = D == 1 ? (ox + 1) * 3 + 1 : o;
            if (!((um >> bit) & 1u))
                continue;
            int xx = x + ox, yy = y + oy;
            if (xx < 0 || xx >= nx)
            {
                if (!g.per0)
                    continue;
                xx = mr_coord(xx, nx, 1);
            }
            if (D == 2 && (yy < 0 || yy >= ny))
            {
                if (!g.per1)
                    continue;
                yy = mr_coord(yy, ny, 1);
            }
            if (fl.kind[li][xy2lin<D>(xx, yy, ny)] & K_INT)
                ib |= 1u << bit;
        }
    const bool fb = (ib & um) || (!g.per0 && (x + ub.x < 0 || x + ub.y >= nx)) ||
                    (D == 2 && !g.per1 && (y + ub.z < 0 || y + ub.w >= ny));
    if (!fb)
        return;
    unsigned mask = 0, dmask = 0;
    for (int pair = 0; pair < 2 * g.q; ++pair)
    {
        const int key = gap * 2 * g.q + pair;
        const int4 db = sdep ? sdep[pair] : aux.tdep[key];
        const bool dom = !((!g.per0 && (x + db.x < 0 || x + db.y >= nx)) || (D == 2 && !g.per1 && (y + db.z < 0 || y + db.w >= ny)));
        const bool ok = dom && !(ib & (spm ? spm[pair] : aux.pmask[key]));
        if (!ok)
            mask |= 1u << pair;
        if (!dom)
            dmask |= 1u << pair;
    }
    // fallback masks live at the value index (read in value-block slot order)
    const int vi = vix<D>(x, y, ny);
    fl.fbm[li][vi] = mask;
    fl.fbd[li][vi] = dmask;
    fl.kind[li][i] = K_LEAF | K_FB;
    // segment lists (thread-per-leaf path): gap-0 fallback leaves and gap-1 leaves whose
    // pairs leave the domain, streamed by K7 MODE 5 / k_fb1 (or MODE 3) from the lists;
    // the other gap-1 leaves are listed tile by tile afterwards (k_list_fb1, MODE 2).
    // One atomic per coalesced group of lanes.
    if (aux.fb1t && (gap == 0 || (gap == 1 && dmask != 0)))
    {
        const int seg = gap == 0 ? 0 : 1;
        const int k = agg_inc(aux.fb_count + 2 + seg, (unsigned)seg);
        if (k < aux.fbs_cap[seg])
            aux.fbs[aux.fbs_off[seg] + k] = (int)i;
        else
            flag_err(aux.err, 2);
    }
    // deep-gap leaves (K8, bands) are listed tile by tile afterwards (k_list_deep)
    if (gap < 2)
    {
        // gap 0 / 1 fallback leaves are found by slot scans (K7 / MODE 2 or k_fb1);
        // count them for the statistics with one atomic per warp
        const unsigned am = __activemask();
        if ((threadIdx.x & 31) == __ffs(am) - 1)
            atomicAdd(aux.fb_count + 1, __popc(am));
    }
}

template <int D>
__global__ void k_fallback(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_, const __grid_constant__ Aux aux)
{
    LSETUP;
    const int li = m - g.J0;
    const int gap = g.J1 - m;
    const int ny = g.ny[li];
    const long long n = (long long)g.nx[li] * ny;
    const int4 ub = aux.udep[gap];
    const int2 pi = aux.upidx[gap];
    LGRID_STRIDE(i, 0, n)
    {
        if (fl.kind[li][i] != K_LEAF)
            continue;
        int x, y;
        lin2xy_l<D>((int)i, ny, g.lny[li], x, y);
        fallback_cell<D>(g, fl, m, li, gap, i, x, y, ub, pi, aux);
    }
}

__global__ void k_fallback_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_, const __grid_constant__ Aux aux)
{
    LSETUP;
    __shared__ int4 sdep[2 * kQ];
    __shared__ unsigned short spm[2 * kQ];
    const int li = m - g.J0;
    const int gap = g.J1 - m;
    for (int t = threadIdx.x; t < 2 * g.q; t += blockDim.x)
    {
        sdep[t] = aux.tdep[gap * 2 * g.q + t];
        spm[t] = aux.pmask[gap * 2 * g.q + t];
    }
    __syncthreads();
    const int ny = g.ny[li];
    const long long nch = (long long)g.nx[li] * ny / 16;
    const int4 ub = aux.udep[gap];
    const int2 pi = aux.upidx[gap];
    LGRID_STRIDE(c, 0, nch)
    {
        V16 k;
        k.v = reinterpret_cast<const uint4*>(fl.kind[li])[c];
        // any byte == K_LEAF (a plain leaf), four bytes per compare
        const unsigned anyw = __vcmpeq4(k.v.x, 0x01010101u * K_LEAF) | __vcmpeq4(k.v.y, 0x01010101u * K_LEAF) |
                              __vcmpeq4(k.v.z, 0x01010101u * K_LEAF) | __vcmpeq4(k.v.w, 0x01010101u * K_LEAF);
        if (!anyw)
            continue;
        const int lin0 = (int)(c * 16);
        const int x = lin0 >> g.lny[li], y0 = lin0 & (ny - 1);
        const int nx = g.nx[li];
        if (aux.umask[gap] == 0)
        {
            // no parent can break the table at this gap (the finest level): only the
            // domain test flags a leaf, so interior chunks are done
            const bool edge = (!g.per0 && (x + ub.x < 0 || x + ub.y >= nx)) ||
                              (!g.per1 && (y0 + ub.z < 0 || y0 + 15 + ub.w >= ny));
            if (!edge)
                continue;
            for (int j = 0; j < 16; ++j)
                if (k.b[j] == K_LEAF)
                    fallback_cell<2>(g, fl, m, li, gap, lin0 + j, x, y0 + j, ub, pi, aux, 0, sdep, spm);
            continue;
        }
        // internal flags of rows x-1, x, x+1 over y0-1 .. y0+16 (clip / wrap)
        uint8_t w[3][18];
#pragma unroll
        for (int r = 0; r < 3; ++r)
        {
            int xr = x + r - 1;
            const bool ok = (xr >= 0 && xr < nx) || g.per0;
            xr = mr_coord(xr, nx, 1);
            V16 v;
            v.v = ok ? reinterpret_cast<const uint4*>(fl.kind[li] + (long long)xr * ny)[y0 >> 4] : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                w[r][j + 1] = ok ? (v.b[j] & K_INT) : 0;
            const int yl = y0 - 1, yr = y0 + 16;
            w[r][0] = (ok && (yl >= 0 || g.per1)) ? (fl.kind[li][(long long)xr * ny + mr_coord(yl, ny, 1)] & K_INT) : 0;
            w[r][17] = (ok && (yr < ny || g.per1)) ? (fl.kind[li][(long long)xr * ny + mr_coord(yr, ny, 1)] & K_INT) : 0;
        }
        for (int j = 0; j < 16; ++j)
            if (k.b[j] == K_LEAF)
            {
                int ib = 0;
#pragma unroll
                for (int o = 0; o < 9; ++o)
                    ib |= (w[o / 3][j + (o % 3)] ? 1 : 0) << o;
                fallback_cell<2>(g, fl, m, li, gap, lin0 + j, x, y0 + j, ub, pi, aux, ib, sdep, spm);
            }
    }
}

// ghost rows: tmp = OR of R membership over y +- 2 (same row)
__global__ void k_ghost_rows_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    const int li = m - g.J0;
    uint8_t* tmp = fl.keep[li];
    const int ny = g.ny[li];
    const long long nch = (long long)g.nx[li] * ny / 16;
    const uint8_t* kind = fl.kind[li];
    LGRID_STRIDE(c, 0, nch)
    {
        const int lin0 = (int)(c * 16);
        const int x = lin0 >> g.lny[li], y0 = lin0 & (ny - 1);
        V16 k, o;
        k.v = reinterpret_cast<const uint4*>(kind)[c];
        uint8_t w[20];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            w[j + 2] = k.b[j] & (K_LEAF | K_INT);
#pragma unroll
        for (int j = 0; j < 2; ++j)
        {
            int yl = y0 - 2 + j, yr = y0 + 16 + j;
            uint8_t vl = 0, vr = 0;
            if (yl >= 0 || g.per1)
                vl = kind[(long long)x * ny + mr_coord(yl, ny, 1)] & (K_LEAF | K_INT);
            if (yr < ny || g.per1)
                vr = kind[(long long)x * ny + mr_coord(yr, ny, 1)] & (K_LEAF | K_INT);
            w[j] = vl;
            w[18 + j] = vr;
        }
        if (ghost_dist(g, m) == 1)
        {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                o.b[j] = w[j + 1] | w[j + 2] | w[j + 3];
        }
        else
        {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                o.b[j] = w[j] | w[j + 1] | w[j + 2] | w[j + 3] | w[j + 4];
        }
        reinterpret_cast<uint4*>(tmp)[c] = o.v;
    }
}

// ghosts: empty cells with an R cell within +-2 rows of tmp
__global__ void k_ghost_v(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    const int li = m - g.J0;
    const uint8_t* tmp = fl.keep[li];
    const int nx = g.nx[li], ny = g.ny[li];
    const long long nch = (long long)nx * ny / 16;
    const int cpr = ny / 16; // chunks per row
    LGRID_STRIDE(c, 0, nch)
    {
        V16 k;
        k.v = reinterpret_cast<const uint4*>(fl.kind[li])[c];
        bool any = false;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            any = any || k.b[j] == 0;
        if (!any)
            continue;
        const int x = (int)(c / cpr), cy = (int)(c - (long long)x * cpr);
        V16 acc;
        acc.v = make_uint4(0, 0, 0, 0);
        const int gd = ghost_dist(g, m);
#pragma unroll
        for (int ox = -2; ox <= 2; ++ox)
        {
            if (ox < -gd || ox > gd)
                continue;
            int xx = x + ox;
            if (xx < 0 || xx >= nx)
            {
                if (!g.per0)
                    continue;
                xx = mr_coord(xx, nx, 1);
            }
            const uint4 t = reinterpret_cast<const uint4*>(tmp)[(long long)xx * cpr + cy];
            acc.v.x |= t.x;
            acc.v.y |= t.y;
            acc.v.z |= t.z;
            acc.v.w |= t.w;
        }
        // byte stores of the marked cells only: the classification (fallback bit on leaf bytes) and
        // the band marking (0 -> K_VIRT) run beside this kernel, and a whole-chunk store of the
        // snapshot would undo theirs
        uint8_t* kb = fl.kind[li] + c * 16;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (k.b[j] == 0 && acc.b[j])
                kb[j] = K_VIRT;
    }
}

// compaction: per-tile counts -> tile scan -> ballot/prefix scatter (lexicographic)
constexpr int kTileThreads = 256;
constexpr int kCellsPerThread = 16;
constexpr int kTile = kTileThreads * kCellsPerThread;

__device__ __forceinline__ int cat_of(uint8_t k)
{
    return (k & K_LEAF) ? 0 : (k & K_INT) ? 1 : (k & K_VIRT) ? 2 : 3;
}

// tile = kTileThreads threads x kCellsPerThread consecutive cells (one 16-byte load each)
__device__ __forceinline__ void load16(const uint8_t* kind, long long base, long long n, uint8_t (&b)[16])
{
    if (base + 16 <= n)
    {
        union {
            uint4 v;
            uint8_t c[16];
        } u;
        u.v = *reinterpret_cast<const uint4*>(kind + base);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            b[j] = u.c[j];
    }
    else
    {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            b[j] = base + j < n ? kind[base + j] : 0;
    }
}

__global__ void __launch_bounds__(kTileThreads) k_tile_count(const uint8_t* kind, long long n, int* tile_counts)
{
    static_assert(kCellsPerThread == 16, "one 16-byte load per thread");
    __shared__ int red[3][kTileThreads / 32];
    const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * 16;
    uint8_t b[16];
    load16(kind, base, n, b);
    // the kinds are exclusive bits: count them four bytes at a time
    int c[3] = {0, 0, 0};
    {
        unsigned wv[4];
        memcpy(wv, b, 16);
#pragma unroll
        for (int k = 0; k < 4; ++k)
        {
            c[0] += __popc(wv[k] & 0x01010101u * K_LEAF);
            c[1] += __popc(wv[k] & 0x01010101u * K_INT);
            c[2] += __popc(wv[k] & 0x01010101u * K_VIRT);
        }
    }
    if (__any_sync(0xffffffffu, (c[0] | c[1] | c[2]) != 0))
    {
        for (int k = 0; k < 3; ++k)
        {
            int v = c[k];
            for (int o = 16; o > 0; o >>= 1)
                v += __shfl_down_sync(0xffffffffu, v, o);
            if ((threadIdx.x & 31) == 0)
                red[k][threadIdx.x >> 5] = v;
        }
    }
    else if ((threadIdx.x & 31) == 0)
    {
        red[0][threadIdx.x >> 5] = 0;
        red[1][threadIdx.x >> 5] = 0;
        red[2][threadIdx.x >> 5] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 3)
    {
        int v = 0;
        for (int w = 0; w < kTileThreads / 32; ++w)
            v += red[threadIdx.x][w];
        tile_counts[(long long)blockIdx.x * 3 + threadIdx.x] = v;
    }
}

// one block: exclusive scan of the tile counts per category, in place; totals -> cnt.
// Per-thread sums of a contiguous tile range, a block-wide exclusive scan of those
// sums (warp shuffles + warp totals in shared memory), then the per-tile offsets.
__device__ __forceinline__ void block_scan_tiles(int* tile_counts, int ntiles, int* cnt)
{
    __shared__ int wsum[3][32];
    const int T = blockDim.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = T >> 5;
    const int per = (ntiles + T - 1) / T;
    const int b = threadIdx.x * per, e = min(ntiles, b + per);
    int loc[3] = {0, 0, 0};
    for (int t = b; t < e; ++t)
        for (int k = 0; k < 3; ++k)
            loc[k] += tile_counts[t * 3 + k];
    int incl[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        int v = loc[k];
        for (int o = 1; o < 32; o <<= 1)
        {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o)
                v += u;
        }
        incl[k] = v;
        if (lane == 31)
            wsum[k][wid] = v;
    }
    __syncthreads();
    if (wid == 0)
    {
#pragma unroll
        for (int k = 0; k < 3; ++k)
        {
            int v = lane < nwarps ? wsum[k][lane] : 0;
            for (int o = 1; o < 32; o <<= 1)
            {
                const int u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o)
                    v += u;
            }
            if (lane < nwarps)
                wsum[k][lane] = v; // inclusive over warps
        }
    }
    __syncthreads();
    int run[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        const int before = wid > 0 ? wsum[k][wid - 1] : 0;
        run[k] = before + incl[k] - loc[k];
        if (threadIdx.x == T - 1)
            cnt[k] = before + incl[k];
    }
    for (int t = b; t < e; ++t)
        for (int k = 0; k < 3; ++k)
        {
            const int v = tile_counts[t * 3 + k];
            tile_counts[t * 3 + k] = run[k];
            run[k] += v;
        }
}

__global__ void k_tile_scan(int* tile_counts, int ntiles, int* cnt)
{
    block_scan_tiles(tile_counts, ntiles, cnt);
}

// per-thread counts of its 16 cells -> block exclusive scan (warp shuffles + warp
// totals in shared memory) -> each thread writes its cells' slots in order:
// lexicographic slots per category
__global__ void __launch_bounds__(kTileThreads) k_tile_scatter(const uint8_t* kind, long long n, const int* tile_offsets,
                                                               const int* cnt, int32_t* map, int32_t* cells)
{
    constexpr int NW = kTileThreads / 32;
    __shared__ int wsum[3][NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * 16;
    uint8_t b[16];
    load16(kind, base, n, b);
    int c[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < 16; ++j)
    {
        c[0] += b[j] & K_LEAF ? 1 : 0;
        c[1] += b[j] & K_INT ? 1 : 0;
        c[2] += b[j] & K_VIRT ? 1 : 0;
    }
    int pre[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        int v = c[k];
        for (int o = 1; o < 32; o <<= 1)
        {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o)
                v += u;
        }
        pre[k] = v - c[k];
        if (lane == 31)
            wsum[k][wid] = v;
    }
    __syncthreads();
    const int catbase[3] = {0, cnt[0], cnt[0] + cnt[1]};
    int pos[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        int wpre = 0;
        for (int w = 0; w < wid; ++w)
            wpre += wsum[k][w];
        pos[k] = catbase[k] + tile_offsets[(long long)blockIdx.x * 3 + k] + wpre + pre[k];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
    {
        const long long i = base + j;
        const int ct = cat_of(b[j]);
        if (i < n && ct < 3)
        {
            const int sl = pos[ct]++;
            if (map)
                map[i] = sl;
            cells[sl] = (int)i;
        }
        else if (i < n && map)
            map[i] = -1;
    }
}

// The step's slot lists are in VALUE-BLOCK order (2D): cells are enumerated by their
// value index vix (sibling blocks, blocks row-major over the parents), so the threads
// of a warp that take consecutive slots touch whole 32-byte value sectors.  The
// slots still hold row-major linear indices; mrlbm_read_leaves re-sorts a level into
// the lexicographic CellIndex order.  (1D: value order == lexicographic order.)
__device__ __forceinline__ bool blk_order(const Geo& g, int li)
{
    return g.d == 2;
}

// row-major linear index of the cell with value index v (2D)
__device__ __forceinline__ int blk_lin(const Geo& g, int li, long long v)
{
    const int ny = g.ny[li], hy = ny >> 1;
    const int G = (int)(v >> 2), c = (int)(v & 3);
    const int gx = G / hy, gy = G - gx * hy;
    return (2 * gx + (c >> 1)) * ny + 2 * gy + (c & 1);
}

// the kinds of value indices [base, base + 16) in value order
__device__ __forceinline__ void load16_blk(const Geo& g, int li, const uint8_t* kind, long long base, long long n,
                                           uint8_t (&b)[16])
{
    if (!blk_order(g, li))
    {
        load16(kind, base, n, b);
        return;
    }
    const int ny = g.ny[li], hy = ny >> 1;
    if ((hy & 3) == 0 && base + 16 <= n)
    {
        // four sibling blocks of one block row: rows 2gx and 2gx + 1, 8 columns each
        const int G = (int)(base >> 2);
        const int gx = G / hy, gy = G - gx * hy;
        union {
            uint2 v;
            uint8_t c[8];
        } r0, r1;
        r0.v = *reinterpret_cast<const uint2*>(kind + (long long)(2 * gx) * ny + 2 * gy);
        r1.v = *reinterpret_cast<const uint2*>(kind + (long long)(2 * gx + 1) * ny + 2 * gy);
#pragma unroll
        for (int k = 0; k < 4; ++k)
        {
            b[4 * k + 0] = r0.c[2 * k];
            b[4 * k + 1] = r0.c[2 * k + 1];
            b[4 * k + 2] = r1.c[2 * k];
            b[4 * k + 3] = r1.c[2 * k + 1];
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
        b[j] = base + j < n ? kind[blk_lin(g, li, base + j)] : 0;
}

// multi-level compaction: block range per level = that level's tiles (count,
// scatter) or one block per level (scan)
__global__ void __launch_bounds__(kTileThreads) k_tile_count_ml(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ TileP tp, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    (void)lvg_;
    const int li = m - g.J0;
    const long long n = g.cap[li];
    const uint8_t* kind = fl.kind[li];
    __shared__ int red[3][kTileThreads / 32];
    const long long base = (long long)lvb_ * kTile + (long long)threadIdx.x * 16;
    uint8_t b[16];
    load16_blk(g, li, kind, base, n, b);
    // the kinds are exclusive bits: count them four bytes at a time
    int c[3] = {0, 0, 0};
    {
        unsigned wv[4];
        memcpy(wv, b, 16);
#pragma unroll
        for (int k = 0; k < 4; ++k)
        {
            c[0] += __popc(wv[k] & 0x01010101u * K_LEAF);
            c[1] += __popc(wv[k] & 0x01010101u * K_INT);
            c[2] += __popc(wv[k] & 0x01010101u * K_VIRT);
        }
    }
    if (__any_sync(0xffffffffu, (c[0] | c[1] | c[2]) != 0))
    {
        for (int k = 0; k < 3; ++k)
        {
            int v = c[k];
            for (int o = 16; o > 0; o >>= 1)
                v += __shfl_down_sync(0xffffffffu, v, o);
            if ((threadIdx.x & 31) == 0)
                red[k][threadIdx.x >> 5] = v;
        }
    }
    else if ((threadIdx.x & 31) == 0)
    {
        red[0][threadIdx.x >> 5] = 0;
        red[1][threadIdx.x >> 5] = 0;
        red[2][threadIdx.x >> 5] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 3)
    {
        int v = 0;
        for (int w = 0; w < kTileThreads / 32; ++w)
            v += red[threadIdx.x][w];
        tp.t[li][(long long)lvb_ * 3 + threadIdx.x] = v;
    }
}

__global__ void k_tile_scan_ml(const __grid_constant__ Geo g, const __grid_constant__ TileP tp, const __grid_constant__ Tree tn, const __grid_constant__ LGrid lg_)
{
    // one block per level; the level totals go to cnt
    LSETUP;
    (void)lvb_;
    (void)lvg_;
    const int li = m - g.J0;
    const int ntiles = (int)((g.cap[li] + kTile - 1) / kTile);
    block_scan_tiles(tp.t[li], ntiles, tn.cnt + li * 4);
}

__global__ void __launch_bounds__(kTileThreads) k_tile_scatter_ml(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const __grid_constant__ TileP tp, const __grid_constant__ Tree tn, const __grid_constant__ LGrid lg_)
{
    LSETUP;
    (void)lvg_;
    const int li = m - g.J0;
    const long long n = g.cap[li];
    const uint8_t* kind = fl.kind[li];
    const int* tile_offsets = tp.t[li];
    const int* cnt = tn.cnt + li * 4;
    int32_t* cells = tn.cells[li];
    constexpr int NW = kTileThreads / 32;
    __shared__ int wsum[3][NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    {
        // empty tile (exclusive offsets equal to the next tile's / the level totals): done
        const int ntl = (int)((n + kTile - 1) / kTile);
        bool empty = true;
        for (int k = 0; k < 3; ++k)
        {
            const int nxt = lvb_ + 1 < ntl ? tile_offsets[(long long)(lvb_ + 1) * 3 + k] : cnt[k];
            empty = empty && nxt == tile_offsets[(long long)lvb_ * 3 + k];
        }
        if (empty)
            return;
    }
    const long long base = (long long)lvb_ * kTile + (long long)threadIdx.x * 16;
    uint8_t b[16];
    load16_blk(g, li, kind, base, n, b);
    const bool blk = blk_order(g, li);
    // the kinds are exclusive bits: count them four bytes at a time
    int c[3] = {0, 0, 0};
    {
        unsigned wv[4];
        memcpy(wv, b, 16);
#pragma unroll
        for (int k = 0; k < 4; ++k)
        {
            c[0] += __popc(wv[k] & 0x01010101u * K_LEAF);
            c[1] += __popc(wv[k] & 0x01010101u * K_INT);
            c[2] += __popc(wv[k] & 0x01010101u * K_VIRT);
        }
    }
    const bool mine = (c[0] | c[1] | c[2]) != 0;
    int pre[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        int v = c[k];
        for (int o = 1; o < 32; o <<= 1)
        {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o)
                v += u;
        }
        pre[k] = v - c[k];
        if (lane == 31)
            wsum[k][wid] = v;
    }
    __syncthreads();
    // the tile's slots are staged in shared memory (category-segmented, lexicographic
    // within each category) and then written out with coalesced stores
    __shared__ int sCells[kTile];
    __shared__ uint8_t sKind[kTile];
    int tot[3], pos[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        int wpre = 0, t = 0;
        for (int w = 0; w < NW; ++w)
        {
            wpre += w < wid ? wsum[k][w] : 0;
            t += wsum[k][w];
        }
        tot[k] = t;
        pos[k] = wpre + pre[k];
    }
    pos[1] += tot[0];
    pos[2] += tot[0] + tot[1];
    if (mine)
    {
        // row-major index of the first cell (block row of 4 sibling blocks when the
        // fast path applies): the others follow by constant offsets, no division per cell
        const int nyl = g.ny[li];
        const bool fast = blk && ((nyl >> 1) & 3) == 0 && base + 16 <= n;
        const int lin0 = fast ? blk_lin(g, li, base) : 0;
#pragma unroll
        for (int j = 0; j < 16; ++j)
        {
            const long long i = base + j;
            const int ct = cat_of(b[j]);
            if (i < n && ct < 3)
            {
                const int sl = pos[ct]++;
                // block k = j / 4, child c = j % 4: (2gx + (c >> 1), 2(gy0 + k) + (c & 1))
                sCells[sl] = fast ? lin0 + ((j & 3) >> 1) * nyl + 2 * (j >> 2) + (j & 1)
                                  : (blk ? blk_lin(g, li, i) : (int)i);
                sKind[sl] = b[j];
            }
        }
    }
    __syncthreads();
    const int catbase[3] = {0, cnt[0], cnt[0] + cnt[1]};
    uint8_t* skind = tn.skind[li];
    int lo = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
    {
        const long long gb = (long long)catbase[k] + tile_offsets[(long long)lvb_ * 3 + k] - lo;
        for (int t = lo + threadIdx.x; t < lo + tot[k]; t += kTileThreads)
        {
            cells[gb + t] = sCells[t];
            skind[gb + t] = sKind[t];
        }
        lo += tot[k];
    }
}

// ---------------------------------------------------------------- K5 transfer, virtual values
// new R cell: old value if it was in the old complete tree (copy / projected),
// else prediction from the new level m-1 values (Decision D.24)
template <int D, int Q>
__global__ void __launch_bounds__(256) k_transfer(const __grid_constant__ Geo g, const __grid_constant__ Tree to, const __grid_constant__ Tree tn, const __grid_constant__ Fld S, int m, const __grid_constant__ Aux aux)
{
    // in place in the state buffer S: cells of the old complete tree keep their value
    // (old leaf / projected internal); cells new to the complete tree are predicted
    // from the (already transferred) new level m-1 values
    const int li = m - g.J0;
    const int nL = tn.cnt[li * 4 + 0], nI = tn.cnt[li * 4 + 1];
    const int ny = g.ny[li];
    const long long cap = g.cap[li];
    GRID_STRIDE(s, 0, nL + nI)
    {
        const int lin = tn.cells[li][s];
        if (to.kind[li][lin] & (K_LEAF | K_INT))
            continue;
        if (m == g.J0)
        {
            flag_err(aux.err, 2);
            continue;
        }
        int x, y;
        lin2xy_l<D>(lin, ny, g.lny[li], x, y);
        const int px = x >> 1, py = y >> 1, dx = x & 1, dy = y & 1;
        constexpr int NS = D == 1 ? 3 : 9;
        int st[NS];
        bool ok = true;
        for (int o = 0; o < NS; ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            ok = ok && (tn.kind[li - 1][mr_lin<D>(g, m - 1, px + ox, py + oy)] & (K_LEAF | K_INT));
            st[o] = mr_vix<D>(g, m - 1, px + ox, py + oy);
        }
        if (!ok)
        {
            flag_err(aux.err, 0);
            continue;
        }
        const long long capp = g.cap[li - 1];
        double v[Q];
#pragma unroll
        for (int h = 0; h < Q; ++h)
        {
            double sv[NS];
            for (int o = 0; o < NS; ++o)
                sv[o] = S.f[li - 1][(long long)h * capp + st[o]];
            v[h] = mr_predict<D>(sv, dx, dy);
        }
        const int vi = vix<D>(x, y, ny);
#pragma unroll
        for (int h = 0; h < Q; ++h)
            S.f[li][(long long)h * cap + vi] = v[h];
    }
}

// virtual cells (ghosts + reconstruction bands): zero-detail prediction from level m-1
template <int D, int Q>
__global__ void __launch_bounds__(256) k_virtual(const __grid_constant__ Geo g, const __grid_constant__ Tree tn, const __grid_constant__ Fld S, int m, const __grid_constant__ Aux aux)
{
    // Virtual slots are in value-block order, so the virtual siblings of one parent are
    // consecutive slots: the first of them (the group leader) loads the parent's stencil
    // once per population and writes every virtual sibling (same mr_predict operands and
    // order as one thread per cell); the other threads of the group return.
    const int li = m - g.J0;
    const int nR = tn.cnt[li * 4 + 0] + tn.cnt[li * 4 + 1], nV = tn.cnt[li * 4 + 2];
    const int ny = g.ny[li];
    const long long cap = g.cap[li], capp = g.cap[li - 1];
    constexpr int NC = 1 << D;
    GRID_STRIDE(s, nR, nR + nV)
    {
        const int lin = tn.cells[li][s];
        int x, y;
        lin2xy_l<D>(lin, ny, g.lny[li], x, y);
        const int px = x >> 1, py = y >> 1;
        if (s > nR)
        {
            int xp, yp;
            lin2xy_l<D>(tn.cells[li][s - 1], ny, g.lny[li], xp, yp);
            if ((xp >> 1) == px && (D == 1 || (yp >> 1) == py))
                continue; // a sibling leads this group
        }
        // the group's virtual cells: children codes c = 2 dx + dy (1D: dx)
        int cc[NC], nc = 0;
        cc[nc++] = D == 1 ? (x & 1) : ((x & 1) << 1) | (y & 1);
        for (int k = 1; k < NC && s + k < nR + nV; ++k)
        {
            int xn, yn;
            lin2xy_l<D>(tn.cells[li][s + k], ny, g.lny[li], xn, yn);
            if ((xn >> 1) != px || (D == 2 && (yn >> 1) != py))
                break;
            cc[nc++] = D == 1 ? (xn & 1) : ((xn & 1) << 1) | (yn & 1);
        }
        constexpr int NS = D == 1 ? 3 : 9;
        int st[NS];
        bool ok = true;
        for (int o = 0; o < NS; ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            ok = ok && tn.kind[li - 1][mr_lin<D>(g, m - 1, px + ox, py + oy)] != 0;
            st[o] = mr_vix<D>(g, m - 1, px + ox, py + oy);
        }
        if (!ok)
        {
            flag_err(aux.err, 0);
            continue;
        }
        // the parent's value block at level m holds the children in code order
        const long long base = D == 1 ? 2LL * px : ((long long)px * (ny >> 1) + py) << 2;
#pragma unroll 3
        for (int h = 0; h < Q; ++h)
        {
            double sv[NS];
#pragma unroll
            for (int o = 0; o < NS; ++o)
                sv[o] = S.f[li - 1][(long long)h * capp + st[o]];
            double* dst = S.f[li] + (long long)h * cap + base;
            for (int k = 0; k < nc; ++k)
            {
                const int c = cc[k];
                dst[c] = mr_predict<D>(sv, D == 1 ? c : c >> 1, D == 1 ? 0 : c & 1);
            }
        }
    }
}

// ---------------------------------------------------------------- K7/K8 stream + collide
// m^eq(conserved moments) with compile-time population indices (EQ = MRLBM_EQ_*).
// Operation order mirrors oracle/mrlbm_oracle.cpp equilibrium() exactly.
template <int EQ, int Q>
__device__ __forceinline__ void equilibrium_t(const double* P, double lambda, const double (&m)[Q], double (&meq)[Q])
{
    if constexpr (EQ == MRLBM_EQ_BURGERS_D1Q2)
    {
        const double u = m[0];
        meq[0] = u;
        meq[1] = __dmul_rn(__dmul_rn(0.5, u), u);
    }
    else if constexpr (EQ == MRLBM_EQ_EULER_D1Q3X3)
    {
        const double gam = P[0];
        const double lam2 = __dmul_rn(lambda, lambda);
        const double rho = m[0], q = m[3], E = m[6];
        const double u = __ddiv_rn(q, rho);
        const double p = __dmul_rn(__dsub_rn(gam, 1.0), __dsub_rn(E, __dmul_rn(__dmul_rn(__dmul_rn(0.5, rho), u), u)));
        const double F[3] = {q, __dadd_rn(__dmul_rn(q, u), p), __dmul_rn(u, __dadd_rn(E, p))};
        const double U[3] = {rho, q, E};
#pragma unroll
        for (int i = 0; i < 3; ++i)
        {
            meq[3 * i + 0] = U[i];
            meq[3 * i + 1] = F[i];
            meq[3 * i + 2] = __dmul_rn(lam2, U[i]);
        }
    }
    else if constexpr (EQ == MRLBM_EQ_ADVECTION_D2Q4)
    {
        const double u = m[0];
        meq[0] = u;
        meq[1] = __dmul_rn(P[0], u);
        meq[2] = __dmul_rn(P[1], u);
        meq[3] = 0.0;
    }
    else if constexpr (EQ == MRLBM_EQ_EULER_D2Q4X4)
    {
        const double gam = P[0];
        const double rho = m[0], qx = m[4], qy = m[8], E = m[12];
        const double u = __ddiv_rn(qx, rho);
        const double v = __ddiv_rn(qy, rho);
        const double ke = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
        const double p = __dmul_rn(__dsub_rn(gam, 1.0), __dsub_rn(E, __dmul_rn(__dmul_rn(0.5, rho), ke)));
        const double Fx[4] = {qx, __dadd_rn(__dmul_rn(qx, u), p), __dmul_rn(qx, v), __dmul_rn(u, __dadd_rn(E, p))};
        const double Fy[4] = {qy, __dmul_rn(qy, u), __dadd_rn(__dmul_rn(qy, v), p), __dmul_rn(v, __dadd_rn(E, p))};
        const double U[4] = {rho, qx, qy, E};
#pragma unroll
        for (int i = 0; i < 4; ++i)
        {
            meq[4 * i + 0] = U[i];
            meq[4 * i + 1] = Fx[i];
            meq[4 * i + 2] = Fy[i];
            meq[4 * i + 3] = 0.0;
        }
    }
    else if constexpr (EQ == MRLBM_EQ_NS_D2Q9)
    {
        const double cs2 = P[0];
        const double rho = m[0], qx = m[1], qy = m[2];
        meq[0] = rho;
        meq[1] = qx;
        meq[2] = qy;
        if (P[1] == 0.0)
        {
            const double q2 = __dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy));
            meq[3] = __dmul_rn(3.0, __dadd_rn(__dmul_rn(__dmul_rn(-2.0, cs2), rho), __ddiv_rn(q2, rho)));
            meq[6] = __dmul_rn(9.0, __dsub_rn(__dmul_rn(__dmul_rn(cs2, cs2), rho), __ddiv_rn(__dmul_rn(cs2, q2), rho)));
        }
        else
        {
            const double qn = __dsqrt_rn(__dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy)));
            meq[3] = __dmul_rn(3.0, __dadd_rn(__dmul_rn(__dmul_rn(-2.0, cs2), rho), __ddiv_rn(qn, rho)));
            meq[6] = __dmul_rn(9.0, __dsub_rn(__dmul_rn(cs2, cs2), __ddiv_rn(__dmul_rn(cs2, qn), rho)));
        }
        meq[4] = __dmul_rn(__dmul_rn(-3.0, cs2), qx);
        meq[5] = __dmul_rn(__dmul_rn(-3.0, cs2), qy);
        meq[7] = __ddiv_rn(__dsub_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy)), rho);
        meq[8] = __ddiv_rn(__dmul_rn(qx, qy), rho);
    }
}

// value of the finest cell (x, y) for the recursive-path E/A sums: inside -> the
// materialised zero-detail reconstruction (leaf or virtual slot at J1); outside
// -> boundary rule by direct evaluation
template <int D>
__device__ __forceinline__ double rim_value(const Geo& g, const Tree& tn, const Fld& S, const SchemeDev* sc, int x,
                                            int y, int h, int leaf_li, long long leaf_lin, const Aux& aux)
{
    const int lj = g.J1 - g.J0;
    const int nx = g.nx[lj], ny = g.ny[lj];
    int face = -1;
    if (!g.per0 && (x < 0 || x >= nx))
        face = x < 0 ? 0 : 1;
    else if (D == 2 && !g.per1 && (y < 0 || y >= ny))
        face = y < 0 ? 2 : 3;
    if (face < 0)
    {
        // the kind and the materialised value are loaded together (the value is
        // speculative: used only when the cell is materialised), one latency
        const int lin = mr_lin<D>(g, g.J1, x, y);
        const uint8_t kself = tn.kind[lj][lin];
        const double vself = S.f[lj][(long long)h * g.cap[lj] + mr_vix<D>(g, g.J1, x, y)];
        if (kself)
            return vself;
        // not materialised (rims of gap-1 leaves): one zero-detail prediction from
        // level J1-1, same operands and order as k_virtual would use; the stencil's
        // kinds and values are again loaded together
        const int lp = lj - 1;
        const int xc = mr_coord(x, nx, g.per0), yc = D == 2 ? mr_coord(y, ny, g.per1) : 0;
        const int px = xc >> 1, py = yc >> 1;
        constexpr int NS = D == 1 ? 3 : 9;
        double sv[NS];
        bool ok = true;
#pragma unroll
        for (int o = 0; o < NS; ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            ok = ok && tn.kind[lp][mr_lin<D>(g, g.J1 - 1, px + ox, py + oy)] != 0;
            sv[o] = S.f[lp][(long long)h * g.cap[lp] + mr_vix<D>(g, g.J1 - 1, px + ox, py + oy)];
        }
        if (!ok)
        {
            flag_err(aux.err, 0);
            return 0.0;
        }
        return mr_predict<D>(sv, xc & 1, yc & 1);
    }
    const int kind = sc->bc_kind[face];
    if (kind == MRLBM_BC_COPY)
    {
        // value of the leaf covering the clamped finest cell: usually the streaming leaf
        // itself (its rim leaves the domain across the face it touches), found without a
        // search; otherwise the covering leaf is searched level by level
        const int cx = mr_coord(x, nx, 0), cy = D == 2 ? mr_coord(y, ny, 0) : 0;
        {
            const int gl = lj - leaf_li;
            int lx, ly;
            lin2xy_l<D>((int)leaf_lin, g.ny[leaf_li], g.lny[leaf_li], lx, ly);
            if ((cx >> gl) == lx && (D == 1 || (cy >> gl) == ly))
                return S.f[leaf_li][(long long)h * g.cap[leaf_li] + vix<D>(lx, ly, g.ny[leaf_li])];
        }
        for (int m = g.J1; m >= g.J0; --m)
        {
            const int li = m - g.J0;
            const int sh = g.J1 - m;
            const int lin = xy2lin<D>(cx >> sh, cy >> sh, g.ny[li]);
            if (tn.kind[li][lin] & K_LEAF)
                return S.f[li][(long long)h * g.cap[li] + vix<D>(cx >> sh, cy >> sh, g.ny[li])];
        }
        flag_err(aux.err, 0);
        return 0.0;
    }
    const int hb = sc->opp[h];
    if (hb < 0)
    {
        flag_err(aux.err, 2);
        return 0.0;
    }
    const double v = S.f[leaf_li][(long long)hb * g.cap[leaf_li] + vl<D>((int)leaf_lin, g.ny[leaf_li], g.lny[leaf_li])];
    if (kind == MRLBM_BC_BOUNCE_BACK)
        return v;
    if (kind == MRLBM_BC_ANTI_BOUNCE_BACK)
        return -v;
    return __dadd_rn(v, sc->bc_add[face][h]);
}

template <int D>
__device__ __forceinline__ bool in_box(int x, int y, int bx0, int bx1, int by0, int by1)
{
    return x >= bx0 && x < bx1 && (D == 1 || (y >= by0 && y < by1));
}

// Sum over the E (side 0) / A (side 1) finest cells in lexicographic order
// (|eta_i| <= 1).  E = (B - eta) \ B, A = B \ (B - eta), enumerated directly:
// full rows where the row leaves B, else the single end column.
template <int D>
__device__ double rim_sum(const Geo& g, const Tree& tn, const Fld& F1, const SchemeDev* sc, int h, int side, int bx0,
                          int bx1, int by0, int by1, int leaf_li, long long leaf_lin, const Aux& aux)
{
    const int ex = sc->eta[h][0], ey = D == 1 ? 0 : sc->eta[h][1];
    double s = 0.0;
    if (ex == 0 && ey == 0)
        return s;
    if (side == 0)
    {
        for (int x = bx0 - ex; x < bx1 - ex; ++x)
        {
            if (x < bx0 || x >= bx1)
            {
                if (D == 1)
                    s = __dadd_rn(s, rim_value<D>(g, tn, F1, sc, x, 0, h, leaf_li, leaf_lin, aux));
                else
                    for (int y = by0 - ey; y < by1 - ey; ++y)
                        s = __dadd_rn(s, rim_value<D>(g, tn, F1, sc, x, y, h, leaf_li, leaf_lin, aux));
            }
            else if (D == 2 && ey != 0)
                s = __dadd_rn(s, rim_value<D>(g, tn, F1, sc, x, ey > 0 ? by0 - 1 : by1, h, leaf_li, leaf_lin, aux));
        }
    }
    else
    {
        for (int x = bx0; x < bx1; ++x)
        {
            if (x + ex < bx0 || x + ex >= bx1)
            {
                if (D == 1)
                    s = __dadd_rn(s, rim_value<D>(g, tn, F1, sc, x, 0, h, leaf_li, leaf_lin, aux));
                else
                    for (int y = by0; y < by1; ++y)
                        s = __dadd_rn(s, rim_value<D>(g, tn, F1, sc, x, y, h, leaf_li, leaf_lin, aux));
            }
            else if (D == 2 && ey != 0)
                s = __dadd_rn(s, rim_value<D>(g, tn, F1, sc, x, ey > 0 ? by1 - 1 : by0, h, leaf_li, leaf_lin, aux));
        }
    }
    return s;
}

// out-of-line rim sum for the rarely taken boundary branch of K7 MODE 3
template <int D>
__device__ __noinline__ double rim_sum_cold(const Geo& g, const Tree& tn, const Fld& F1, const SchemeDev* sc, int h,
                                            int side, int bx0, int bx1, int by0, int by1, int leaf_li,
                                            long long leaf_lin, const Aux& aux)
{
    return rim_sum<D>(g, tn, F1, sc, h, side, bx0, bx1, by0, by1, leaf_li, leaf_lin, aux);
}

// the boundary rim sum of a gap-1 leaf as a by-value functor (params by address:
// __grid_constant__, no copies)
template <int D>
struct RimCold {
    const Geo* g;
    const Tree* tn;
    const Fld* F1;
    const SchemeDev* sc;
    const Aux* aux;
    int x, y, li, lin;
    __device__ __forceinline__ double operator()(int h, int side) const
    {
        return rim_sum_cold<D>(*g, *tn, *F1, sc, h, side, 2 * x, 2 * x + 2, D == 1 ? 0 : 2 * y, D == 1 ? 1 : 2 * y + 2,
                               li, lin, *aux);
    }
};

// The i-th finest-level cell of the E (side 0) or A (side 1) rim of the box
// [bx0, bx1) x [by0, by1) for velocity (ex, ey), in rim_sum's loop order: at most one
// x of the range contributes a whole column (the first or the last), the others one
// cell each when ey != 0.  Returns the count with i < 0.
template <int D>
__device__ __forceinline__ int rim_cell(int side, int ex, int ey, int bx0, int bx1, int by0, int by1, int i, int& x,
                                        int& y)
{
    const int nx = bx1 - bx0;
    const int colLen = D == 2 ? by1 - by0 : 1;
    const bool single = D == 2 && ey != 0;
    // column position: 0 none, 1 first x of the range, 2 last
    const int colpos = ex == 0 ? 0 : (side == 0 ? (ex > 0 ? 1 : 2) : (ex > 0 ? 2 : 1));
    const int xs = side == 0 ? bx0 - ex : bx0;
    const int ycol = side == 0 ? by0 - ey : by0;
    const int ysgl = side == 0 ? (ey > 0 ? by0 - 1 : by1) : (ey > 0 ? by1 - 1 : by0);
    const int nsg = single ? nx - (colpos ? 1 : 0) : 0;
    if (i < 0)
        return (colpos ? colLen : 0) + nsg;
    if (colpos == 1)
    {
        if (i < colLen)
        {
            x = xs;
            y = D == 2 ? ycol + i : 0;
        }
        else
        {
            x = xs + 1 + (i - colLen);
            y = ysgl;
        }
    }
    else if (colpos == 2)
    {
        if (i < nsg)
        {
            x = xs + i;
            y = ysgl;
        }
        else
        {
            x = xs + nx - 1;
            y = D == 2 ? ycol + (i - nsg) : 0;
        }
    }
    else
    {
        x = xs + i;
        y = ysgl;
    }
    return 0;
}

// K8: stream of the deep-gap (gap >= 2) fallback leaves, one warp per (leaf,
// population).  Each side uses the flattened table when it is exact for this leaf,
// else the recursive reconstruction of the finest-level rim (materialised band cells
// or on-the-fly predictions, plus the boundary rule).  The lanes load the table
// operands / evaluate the rim cells in parallel; the sums are then accumulated in
// table / rim order through shuffles, so the arithmetic is rim_sum's.  Writes
// post-stream populations into F0; K7 collides them.
template <int D>
__global__ void __launch_bounds__(256, 4) k_stream_fallback(const __grid_constant__ Geo g, const __grid_constant__ Tree tn, const __grid_constant__ Fld F0, const __grid_constant__ Fld F1, const __grid_constant__ Flags fl, const SchemeDev* sc,
                                                         Aux aux)
{
    const int nfb = min(*aux.fb_count, (int)aux.fb_cap);
    const int q = g.q;
    const int lane = threadIdx.x & 31;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long t = gw; t < (long long)nfb * q; t += nw)
    {
        const int it = (int)(t / q), h = (int)(t % q);
        const int2 e = aux.fb_list[it];
        if (g.J1 - e.x < 2)
            continue; // gap 1: k_fb1
        const unsigned mask = aux.fb_mask[it];
        const int m = e.x, li = m - g.J0;
        const long long slot = e.y; // dense storage: values live at the linear index
        const int ny = g.ny[li];
        const long long cap = g.cap[li];
        int x, y;
        lin2xy_l<D>(e.y, ny, g.lny[li], x, y);
        const int gap = g.J1 - m;
        const int ex = sc->eta[h][0], ey = D == 1 ? 0 : sc->eta[h][1];
        double sums[2];
        for (int side = 0; side < 2; ++side)
        {
            double acc = 0.0;
            if (((mask >> (2 * h + side)) & 1u) == 0)
            {
                // flattened table (<= 25 entries): one operand per lane, summed in order
                const int2 ti = aux.tidx[(gap * q + h) * 2 + side];
                for (int b0 = 0; b0 < ti.y; b0 += 32)
                {
                    double v = 0.0;
                    if (b0 + lane < ti.y)
                    {
                        const int k = ti.x + b0 + lane;
                        const int2 o = aux.toff[k];
                        const int sl = mr_lin<D>(g, m, x + o.x, y + o.y);
                        if (!tn.kind[li][sl])
                            flag_err(aux.err, 0);
                        v = __dmul_rn(aux.tw[k], F1.f[li][(long long)h * cap + mr_vix<D>(g, m, x + o.x, y + o.y)]);
                    }
                    const int nv = min(32, ti.y - b0);
                    for (int j = 0; j < nv; ++j)
                        acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, v, j));
                }
            }
            else if (ex != 0 || ey != 0)
            {
                const int side_n = 1 << gap;
                const int bx0 = x * side_n, bx1 = bx0 + side_n;
                const int by0 = D == 1 ? 0 : y * side_n, by1 = D == 1 ? 1 : by0 + side_n;
                int xr = 0, yr = 0;
                const int n = rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, -1, xr, yr);
                for (int b0 = 0; b0 < n; b0 += 32)
                {
                    double v = 0.0;
                    if (b0 + lane < n)
                    {
                        rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, b0 + lane, xr, yr);
                        v = rim_value<D>(g, tn, F1, sc, xr, yr, h, li, slot, aux);
                    }
                    const int nv = min(32, n - b0);
                    for (int j = 0; j < nv; ++j)
                        acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, v, j));
                }
            }
            sums[side] = acc;
        }
        if (lane == 0)
        {
            const double scale = ldexp(1.0, D * (m - g.J1));
            const long long o = (long long)h * cap + vix<D>(x, y, ny);
            F0.f[li][o] = __dadd_rn(F1.f[li][o], __dmul_rn(scale, __dsub_rn(sums[0], sums[1])));
        }
    }
}

// K8 (default): the same stream of the deep-gap fallback leaves, one THREAD per (leaf,
// population).  Each side's sum is accumulated serially in table / rim order from 0.0,
// exactly rim_sum's arithmetic (and the warp kernel's), but 32 independent sums run per
// warp instead of one, so no lane idles on short rims (4..2^(gap+1) cells) and no
// shuffle chain serialises the adds.  Rim cells are fetched in batches of kRimB: the
// kinds and the (speculative) materialised values of a batch are loaded together so
// kRimB independent loads are in flight per thread; cells outside the domain or not
// materialised take the general rim_value path.
constexpr int kRimB = 8;
// leaves with gap >= kLongGap (rims of 2^gap .. 2^(gap+1) finest cells per side) go to the
// warp-cooperative K8 launch instead of one thread per (leaf, population)

// Finest-level rim sum of a deep-gap leaf (2D), the finest rim cells reconstructed on the
// fly: a cell in R (a finest leaf) contributes its value; any other cell inside the
// domain contributes the zero-detail prediction from its parent's 3 x 3 stencil at level
// J1-1 -- the value k_virtual would have materialised there (same mr_predict operands
// and order), so the sum is bit-identical to summing a materialised finest band.  The
// rim is at most two straight segments (a column and a row, rim_cell's order); along a
// segment consecutive cells share their parent or move it by one, so the stencil is a
// sliding 3 x 3 window (3 new values per parent instead of 9 per cell).  Cells outside a
// non-periodic domain take the boundary rule (rim_value).
struct StencilWin {
    double v[9];
    int px = INT_MIN, py = INT_MIN;
};

// (The window lives in local memory, indexed at run time: measured faster than a
// register window with compile-time indices, 0.88 vs 1.66-1.96 ms per window step --
// the register version cost 43 more registers or spilled under a bound.)
template <int D>
__device__ __forceinline__ void win_load(const Geo& g, const Tree& tn, const double* fp, StencilWin& w, int px, int py,
                                         const Aux& aux)
{
    const int lp = g.nlev - 2, mp = g.J1 - 1;
    int o0 = 0, o1 = 9; // stencil entries to load
    int step = 1;
    if (px == w.px && py == w.py + 1)
    {
        // column slide: shift oy, load the oy = +1 entries
#pragma unroll
        for (int ox = 0; ox < 3; ++ox)
        {
            w.v[ox * 3 + 0] = w.v[ox * 3 + 1];
            w.v[ox * 3 + 1] = w.v[ox * 3 + 2];
        }
        o0 = 2;
        step = 3;
    }
    else if (py == w.py && px == w.px + 1)
    {
        // row slide: shift ox, load the ox = +1 entries
#pragma unroll
        for (int oy = 0; oy < 3; ++oy)
        {
            w.v[0 * 3 + oy] = w.v[1 * 3 + oy];
            w.v[1 * 3 + oy] = w.v[2 * 3 + oy];
        }
        o0 = 6;
    }
    else if (px == w.px && py == w.py)
        return;
    bool ok = true;
    for (int o = o0; o < o1; o += step)
    {
        const int ox = o / 3 - 1, oy = o % 3 - 1;
        ok = ok && tn.kind[lp][mr_lin<D>(g, mp, px + ox, py + oy)] != 0;
        w.v[o] = fp[mr_vix<D>(g, mp, px + ox, py + oy)];
    }
    if (!ok)
        flag_err(aux.err, 0);
    w.px = px;
    w.py = py;
}

template <int D>
__device__ double rim_sum_j1(const Geo& g, const Tree& tn, const Fld& F1, const SchemeDev* sc, int h, int side, int ex,
                             int ey, int bx0, int bx1, int by0, int by1, int leaf_li, long long leaf_lin, const Aux& aux)
{
    const int lj = g.nlev - 1;
    const int nxf = g.nx[lj], nyf = g.ny[lj];
    const double* ff = F1.f[lj] + (long long)h * g.cap[lj];
    const double* fp = F1.f[lj - 1] + (long long)h * g.cap[lj - 1];
    int xr = 0, yr = 0;
    const int n = rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, -1, xr, yr);
    StencilWin w;
    double acc = 0.0;
#pragma unroll 1
    for (int i = 0; i < n; ++i)
    {
        int cx, cy;
        rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, i, cx, cy);
        const bool inside = (g.per0 || (cx >= 0 && cx < nxf)) && (g.per1 || (cy >= 0 && cy < nyf));
        double val;
        if (!inside)
            val = rim_value<D>(g, tn, F1, sc, cx, cy, h, leaf_li, leaf_lin, aux);
        else
        {
            const int xc = mr_coord(cx, nxf, g.per0), yc = mr_coord(cy, nyf, g.per1);
            const int lin = xc * nyf + yc;
            if (tn.kind[lj][lin] & K_LEAF)
                val = ff[vix<D>(xc, yc, nyf)];
            else
            {
                win_load<D>(g, tn, fp, w, xc >> 1, yc >> 1, aux);
                val = mr_predict<D>(w.v, xc & 1, yc & 1);
            }
        }
        acc = __dadd_rn(acc, val);
    }
    return acc;
}

template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) k_stream_fallback_t(const __grid_constant__ Geo g, const __grid_constant__ Tree tn,
                                                              const __grid_constant__ Fld F0, const __grid_constant__ Fld F1,
                                                              const SchemeDev* sc, const __grid_constant__ Aux aux)
{
    const int nfb = min(*aux.fb_count, (int)aux.fb_cap);
    const int q = g.q;
    const int lj = g.J1 - g.J0;
    const int nxf = g.nx[lj], nyf = g.ny[lj];
    const long long capf = g.cap[lj];
    // task t: chunk of 32 list entries x q populations; a warp = one population of the
    // chunk's 32 (spatially neighbouring) leaves, so the warp's lanes take the same side
    // path together.  (Splitting the two sides over a lane pair diverged on every leaf
    // with one table side and one rim side: measured 1.53 vs 0.88 ms per window step.)
    const long long nchunk = ((long long)nfb + 31) / 32;
    const int long_gap = k8_long_gap(aux.k8_long, aux.fb_count);
    GRID_STRIDE(t, 0, nchunk * 32 * q)
    {
        const long long chunk = t / (32 * q);
        const int r = (int)(t - chunk * 32 * q);
        const int h = r >> 5;
        const int it = (int)(chunk * 32 + (r & 31));
        if (it >= nfb)
            continue;
        const int2 e = aux.fb_list[it];
        const int m = e.x;
        const int gap = g.J1 - m;
        if (gap < 2 || (long_gap > 0 && gap >= long_gap))
            continue; // gap 0 / 1: K7 MODE 2 / 5 and k_fb1; long rims: k_stream_fallback_long
        const unsigned mask = aux.fb_mask[it];
        const int li = m - g.J0;
        const int ny = g.ny[li];
        const long long cap = g.cap[li];
        int x, y;
        lin2xy_l<D>(e.y, ny, g.lny[li], x, y);
        const int ex = sc->eta[h][0], ey = D == 1 ? 0 : sc->eta[h][1];
        double sum_e = 0.0, sum_a = 0.0; // scalars: an indexed array would live on the stack
#pragma unroll 1
        for (int side = 0; side < 2; ++side)
        {
            double acc = 0.0;
            if (((mask >> (2 * h + side)) & 1u) == 0)
            {
                // flattened table, in table order
                const int2 ti = aux.tidx[(gap * q + h) * 2 + side];
                const double* fm = F1.f[li] + (long long)h * cap;
#pragma unroll 1
                for (int k0 = 0; k0 < ti.y; k0 += kRimB)
                {
                    double v[kRimB];
#pragma unroll
                    for (int j = 0; j < kRimB; ++j)
                    {
                        v[j] = 0.0;
                        if (k0 + j < ti.y)
                        {
                            const int k = ti.x + k0 + j;
                            const int2 o = aux.toff[k];
                            // (no kind check: the table offsets stay inside the 5^D box, which the ghost
                            // layer materialises around every R cell, ghost_dist = 2 below the finest
                            // level; K7's table path does not check either)
                            v[j] = __dmul_rn(aux.tw[k], fm[mr_vix<D>(g, m, x + o.x, y + o.y)]);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kRimB; ++j)
                        if (k0 + j < ti.y)
                            acc = __dadd_rn(acc, v[j]);
                }
            }
            else if (D == 2 && (ex != 0 || ey != 0))
            {
                const int side_n = 1 << gap;
                const int bx0 = x * side_n, by0 = y * side_n;
                acc = rim_sum_j1<D>(g, tn, F1, sc, h, side, ex, ey, bx0, bx0 + side_n, by0, by0 + side_n, li, e.y, aux);
            }
            else if (ex != 0 || ey != 0)
            {
                const int side_n = 1 << gap;
                const int bx0 = x * side_n, bx1 = bx0 + side_n;
                const int by0 = D == 1 ? 0 : y * side_n, by1 = D == 1 ? 1 : by0 + side_n;
                int xr = 0, yr = 0;
                const int n = rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, -1, xr, yr);
                const double* ff = F1.f[lj] + (long long)h * capf;
#pragma unroll 1
                for (int i = 0; i < n; ++i)
                {
                    int cx, cy;
                    rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, i, cx, cy);
                    const bool inside = (g.per0 || (cx >= 0 && cx < nxf)) && (D == 1 || g.per1 || (cy >= 0 && cy < nyf));
                    const uint8_t kd = inside ? tn.kind[lj][mr_lin<D>(g, g.J1, cx, cy)] : 0;
                    const double w = kd ? ff[mr_vix<D>(g, g.J1, cx, cy)]
                                        : rim_value<D>(g, tn, F1, sc, cx, cy, h, li, e.y, aux);
                    acc = __dadd_rn(acc, w);
                }
            }
            if (side == 0)
                sum_e = acc;
            else
                sum_a = acc;
        }
        const double scale = ldexp(1.0, D * (m - g.J1));
        const long long o = (long long)h * cap + vix<D>(x, y, ny);
        F0.f[li][o] = __dadd_rn(F1.f[li][o], __dmul_rn(scale, __dsub_rn(sum_e, sum_a)));
    }
}

// K8, long rims (gap >= kLongGap): one warp per (leaf, population) over the tail list of
// k_list_deep.  A thread-per-(leaf, population) chain over 2^gap .. 2^(gap+1) rim cells
// (up to 2 x 512 dependent fetch-predict-add rounds at gap 8) set the duration of the
// whole K8 launch in the settled and developing regimes, where such leaves are few.  Here
// the lanes evaluate 32 rim cells (or load 32 table operands) at a time into shared
// memory and lane 0 accumulates them serially in rim / table order from 0.0: the same
// operands and the same order of additions as rim_sum, so bit-identical.
template <int D>
__global__ void __launch_bounds__(256) k_stream_fallback_long(const __grid_constant__ Geo g, const __grid_constant__ Tree tn,
                                                                 const __grid_constant__ Fld F0, const __grid_constant__ Fld F1,
                                                                 const SchemeDev* sc, const __grid_constant__ Aux aux)
{
    __shared__ double sv[8][32];
    const int nlong = aux.fb_count[5];
    const int long_gap = k8_long_gap(aux.k8_long, aux.fb_count);
    const int q = g.q;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    if (long_gap > aux.k8_long && aux.fb_count[6] == 0)
        return; // many long-rim leaves, none at the raised threshold: all of them are the thread kernel's
    for (long long t = gw; t < (long long)nlong * q; t += nw)
    {
        const int2 te = aux.fb_list[aux.fb_cap - 1 - (t / q)]; // (index into the list, level)
        if (g.J1 - te.y < long_gap)
            continue; // many long-rim leaves this step: the thread kernel takes this gap
        const int it = te.x, h = (int)(t % q);
        const int2 e = aux.fb_list[it];
        const unsigned mask = aux.fb_mask[it];
        const int m = e.x, li = m - g.J0;
        const int ny = g.ny[li];
        const long long cap = g.cap[li];
        int x, y;
        lin2xy_l<D>(e.y, ny, g.lny[li], x, y);
        const int gap = g.J1 - m;
        const int ex = sc->eta[h][0], ey = D == 1 ? 0 : sc->eta[h][1];
        double sum_e = 0.0, sum_a = 0.0;
        for (int side = 0; side < 2; ++side)
        {
            double acc = 0.0;
            const bool table = ((mask >> (2 * h + side)) & 1u) == 0;
            int n = 0;
            int2 ti = make_int2(0, 0);
            const int side_n = 1 << gap;
            const int bx0 = x * side_n, bx1 = bx0 + side_n;
            const int by0 = D == 1 ? 0 : y * side_n, by1 = D == 1 ? 1 : by0 + side_n;
            if (table)
            {
                ti = aux.tidx[(gap * q + h) * 2 + side];
                n = ti.y;
            }
            else if (ex != 0 || ey != 0)
            {
                int xr = 0, yr = 0;
                n = rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, -1, xr, yr);
            }
            for (int b0 = 0; b0 < n; b0 += 32)
            {
                double v = 0.0;
                if (b0 + lane < n)
                {
                    if (table)
                    {
                        const int k = ti.x + b0 + lane;
                        const int2 o = aux.toff[k];
                        if (!tn.kind[li][mr_lin<D>(g, m, x + o.x, y + o.y)])
                            flag_err(aux.err, 0);
                        v = __dmul_rn(aux.tw[k], F1.f[li][(long long)h * cap + mr_vix<D>(g, m, x + o.x, y + o.y)]);
                    }
                    else
                    {
                        int xr = 0, yr = 0;
                        rim_cell<D>(side, ex, ey, bx0, bx1, by0, by1, b0 + lane, xr, yr);
                        v = rim_value<D>(g, tn, F1, sc, xr, yr, h, li, e.y, aux);
                    }
                }
                sv[w][lane] = v;
                __syncwarp();
                if (lane == 0)
                {
                    const int nv = min(32, n - b0);
                    for (int j = 0; j < nv; ++j)
                        acc = __dadd_rn(acc, sv[w][j]);
                }
                __syncwarp();
            }
            if (side == 0)
                sum_e = acc;
            else
                sum_a = acc;
        }
        if (lane == 0)
        {
            const double scale = ldexp(1.0, D * (m - g.J1));
            const long long o = (long long)h * cap + vix<D>(x, y, ny);
            F0.f[li][o] = __dadd_rn(F1.f[li][o], __dmul_rn(scale, __dsub_rn(sum_e, sum_a)));
        }
    }
}

// K8 variant (MRLBM_K8_BLOCK=1): the same stream, one block per chunk of 32 consecutive list entries
// (spatial neighbours, k_list_deep) with one warp per population (blockDim = 32 q), one
// thread per (leaf, population).  The value indices of each leaf's distinct table
// offsets (<= 5^D box cells, with the MR clamp / wrap and the resolved-stencil check)
// are computed once per leaf into shared memory instead of once per table entry and
// population, so a table sum costs a shared index load, a value load and the fp ops
// per entry.  Sums stay serial in table / rim order from 0.0 (bit-identical).
template <int D>
__global__ void __launch_bounds__(512) k_stream_fallback_b(const __grid_constant__ Geo g, const __grid_constant__ Tree tn,
                                                           const __grid_constant__ Fld F0, const __grid_constant__ Fld F1,
                                                           const SchemeDev* sc, const __grid_constant__ Aux aux)
{
    constexpr int kU = D == 1 ? 5 : 25;
    __shared__ int sBox[32][kU + 1];
    __shared__ int2 sLeaf[32];
    __shared__ unsigned sMask[32];
    const int nfb = min(*aux.fb_count, (int)aux.fb_cap);
    const int q = g.q;
    const int lane = threadIdx.x & 31, h = threadIdx.x >> 5;
    const int nchunk = (nfb + 31) / 32;
    for (int c = blockIdx.x; c < nchunk; c += gridDim.x)
    {
        if (threadIdx.x < 32)
        {
            const int it = c * 32 + threadIdx.x;
            sLeaf[threadIdx.x] = it < nfb ? aux.fb_list[it] : make_int2(-1, 0);
            sMask[threadIdx.x] = it < nfb ? aux.fb_mask[it] : 0u;
        }
        __syncthreads();
        for (int k = threadIdx.x; k < 32 * kU; k += blockDim.x)
        {
            const int i = k / kU, u = k - i * kU;
            const int2 e = sLeaf[i];
            if (e.x < 0)
                continue;
            const int2 gu = aux.guidx[g.J1 - e.x];
            if (u >= gu.y)
                continue;
            const int2 o = aux.guoff[gu.x + u];
            const int li = e.x - g.J0;
            int x, y;
            lin2xy_l<D>(e.y, g.ny[li], g.lny[li], x, y);
            if (!tn.kind[li][mr_lin<D>(g, e.x, x + o.x, y + o.y)])
                flag_err(aux.err, 0);
            sBox[i][u] = mr_vix<D>(g, e.x, x + o.x, y + o.y);
        }
        __syncthreads();
        const int2 e = sLeaf[lane];
        const int m = e.x;
        if (m >= 0 && g.J1 - m >= 2)
        {
            const int gap = g.J1 - m;
            const unsigned mask = sMask[lane];
            const int li = m - g.J0;
            const int ny = g.ny[li];
            const long long cap = g.cap[li];
            int x, y;
            lin2xy_l<D>(e.y, ny, g.lny[li], x, y);
            const int ex = sc->eta[h][0], ey = D == 1 ? 0 : sc->eta[h][1];
            const double* fm = F1.f[li] + (long long)h * cap;
            double sum_e = 0.0, sum_a = 0.0;
#pragma unroll 1
            for (int side = 0; side < 2; ++side)
            {
                double acc = 0.0;
                if (((mask >> (2 * h + side)) & 1u) == 0)
                {
                    // flattened table, in table order
                    const int2 ti = aux.tidx[(gap * q + h) * 2 + side];
#pragma unroll 1
                    for (int k0 = 0; k0 < ti.y; k0 += kRimB)
                    {
                        double v[kRimB];
#pragma unroll
                        for (int j = 0; j < kRimB; ++j)
                            v[j] = k0 + j < ti.y ? __dmul_rn(aux.tw[ti.x + k0 + j], fm[sBox[lane][aux.tu[ti.x + k0 + j]]])
                                                 : 0.0;
#pragma unroll
                        for (int j = 0; j < kRimB; ++j)
                            if (k0 + j < ti.y)
                                acc = __dadd_rn(acc, v[j]);
                    }
                }
                else if (ex != 0 || ey != 0)
                {
                    const int side_n = 1 << gap;
                    const int bx0 = x * side_n, bx1 = bx0 + side_n;
                    const int by0 = D == 1 ? 0 : y * side_n, by1 = D == 1 ? 1 : by0 + side_n;
                    if constexpr (D == 2)
                        acc = rim_sum_j1<D>(g, tn, F1, sc, h, side, ex, ey, bx0, bx1, by0, by1, li, e.y, aux);
                    else
                        acc = rim_sum<D>(g, tn, F1, sc, h, side, bx0, bx1, by0, by1, li, e.y, aux);
                }
                if (side == 0)
                    sum_e = acc;
                else
                    sum_a = acc;
            }
            const double scale = ldexp(1.0, D * (m - g.J1));
            const long long o = (long long)h * cap + vix<D>(x, y, ny);
            F0.f[li][o] = __dadd_rn(F1.f[li][o], __dmul_rn(scale, __dsub_rn(sum_e, sum_a)));
        }
        __syncthreads();
    }
}

// config 5 volume-fraction blend: the fraction alpha
// of the cell (level m, index x, y) inside the disc, from ns x ns sub-samples; 0 when
// the cell's box misses the disc's bounding box.
__device__ __forceinline__ double obstacle_alpha(const SchemeDev* scg, int m, int x, int y)
{
    const double dx = ldexp(1.0, -m);
    const double ox = scg->origin[0], oy = scg->origin[1];
    const double cx = scg->obs_c[0], cy = scg->obs_c[1], r = scg->obs_r;
    const double x0 = __dadd_rn(ox, __dmul_rn((double)x, dx));
    const double y0 = __dadd_rn(oy, __dmul_rn((double)y, dx));
    const double x1 = __dadd_rn(x0, dx), y1 = __dadd_rn(y0, dx);
    if (x1 < __dsub_rn(cx, r) || x0 > __dadd_rn(cx, r) || y1 < __dsub_rn(cy, r) || y0 > __dadd_rn(cy, r))
        return 0.0;
    const int ns = scg->obs_ns;
    const double r2 = __dmul_rn(r, r);
    int cnt = 0;
    for (int a = 0; a < ns; ++a)
    {
        const double sx = __dadd_rn(ox, __dmul_rn(__dadd_rn((double)x, __ddiv_rn((double)a + 0.5, (double)ns)), dx));
        const double ddx = __dsub_rn(sx, cx);
        const double rx = __dmul_rn(ddx, ddx);
        for (int b = 0; b < ns; ++b)
        {
            const double sy = __dadd_rn(oy, __dmul_rn(__dadd_rn((double)y, __ddiv_rn((double)b + 0.5, (double)ns)), dx));
            const double ddy = __dsub_rn(sy, cy);
            cnt += __dadd_rn(rx, __dmul_rn(ddy, ddy)) < r2;
        }
    }
    return cnt > 0 ? __ddiv_rn((double)cnt, (double)(ns * ns)) : 0.0;
}

// alpha of a leaf from the table built at create (k_alpha_table: obstacle_alpha of every
// cell of the per-level boxes around the disc), 0 outside the box: the geometry is
// static, so the hot kernels do one load instead of 16 x 16 sub-samples per step
__device__ __forceinline__ double obstacle_alpha_cached(const Aux& aux, int li, int x, int y)
{
    const int bx = x - aux.frc_x0[li], by = y - aux.frc_y0[li];
    if (bx < 0 || by < 0 || bx >= aux.frc_nx[li] || by >= aux.frc_ny[li])
        return 0.0;
    return aux.alpha_tab[(aux.frc_off[li] >> 1) + (long long)bx * aux.frc_ny[li] + by];
}

__global__ void k_alpha_table(const SchemeDev* scg, int m, int x0, int y0, int nx, int ny, double* out)
{
    GRID_STRIDE(i, 0, (long long)nx * ny)
    {
        const int bx = (int)(i / ny), by = (int)(i - (long long)bx * ny);
        out[i] = obstacle_alpha(scg, m, x0 + bx, y0 + by);
    }
}

// obstacle force term of one leaf (oracle force_terms): the momentum the blend removes
// per unit time, alpha * q * |cell| / dt, q = post-collision momentum moments mo[1..2]
__device__ __forceinline__ void force_store(const Aux& aux, const Geo& g, const SchemeDev* scg, int m, int x, int y,
                                         double alpha, double mx, double my)
{
    const int li = m - g.J0;
    const int bx = x - aux.frc_x0[li], by = y - aux.frc_y0[li];
    if (bx < 0 || by < 0 || bx >= aux.frc_nx[li] || by >= aux.frc_ny[li])
    {
        flag_err(aux.err, 2);
        return;
    }
    const double area = ldexp(1.0, -2 * m);
    const double dt = __ddiv_rn(ldexp(1.0, -g.J1), scg->lambda);
    double* o = aux.frc + aux.frc_off[li] + 2LL * ((long long)bx * aux.frc_ny[li] + by);
    o[0] = __ddiv_rn(__dmul_rn(__dmul_rn(alpha, mx), area), dt);
    o[1] = __ddiv_rn(__dmul_rn(__dmul_rn(alpha, my), area), dt);
}

// deterministic sum of the force boxes (level by level, fixed strided partition and
// tree): appends (Fx, Fy) of this step to the history; one block of 1024 threads
__global__ void __launch_bounds__(1024) k_force_sum(const double* frc, long long n, double* hist, int* hn, int cap)
{
    __shared__ double s0[1024], s1[1024];
    double a0 = 0.0, a1 = 0.0;
    for (long long i = threadIdx.x; i < n; i += 1024)
    {
        a0 = __dadd_rn(a0, frc[2 * i]);
        a1 = __dadd_rn(a1, frc[2 * i + 1]);
    }
    s0[threadIdx.x] = a0;
    s1[threadIdx.x] = a1;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1)
    {
        if ((int)threadIdx.x < w)
        {
            s0[threadIdx.x] = __dadd_rn(s0[threadIdx.x], s0[threadIdx.x + w]);
            s1[threadIdx.x] = __dadd_rn(s1[threadIdx.x], s1[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
    {
        const int k = *hn;
        if (k < cap)
        {
            hist[2 * k] = s0[0];
            hist[2 * k + 1] = s1[0];
        }
        *hn = k + 1;
    }
}

// generated unrolled table sums (stream_gen.cuh) for the built-in velocity sets
// GC: gap class compiled in (0: gap 0 only, 1: gaps >= 1 only, -1: any)
template <int EQ, int Q, int GC>
__device__ __forceinline__ void gen_stream(int gap, const double* Fin, long long cap, int x, int y, int nx, int ny,
                                           int per0, int per1, long long s, const double* sW, double scale,
                                           double (&f)[Q])
{
#define GEN_CALL(N)                                                                                                    \
    if constexpr (GC == 0)                                                                                             \
        gen_stream_EQ##N##_g0(Fin, cap, x, y, nx, ny, per0, per1, s, sW, scale, f);                               \
    else                                                                                                               \
    {                                                                                                                  \
        if (GC < 0 && gap == 0)                                                                                        \
            gen_stream_EQ##N##_g0(Fin, cap, x, y, nx, ny, per0, per1, s, sW, scale, f);                           \
        else if (gap == 1)                                                                                             \
            gen_stream_EQ##N##_g1(Fin, cap, x, y, nx, ny, per0, per1, s, sW, scale, f);                           \
        else                                                                                                           \
            gen_stream_EQ##N##_g2(Fin, cap, x, y, nx, ny, per0, per1, s, sW, scale, f);                           \
    }
    if constexpr (EQ == 1 && Q == 2)
    {
        GEN_CALL(1)
    }
    else if constexpr (EQ == 2 && Q == 9)
    {
        GEN_CALL(2)
    }
    else if constexpr (EQ == 3 && Q == 4)
    {
        GEN_CALL(3)
    }
    else if constexpr (EQ == 4 && Q == 16)
    {
        GEN_CALL(4)
    }
    else if constexpr (EQ == 5 && Q == 9)
    {
        GEN_CALL(5)
    }
#undef GEN_CALL
}

// the scheme's matrices as a kernel parameter (constant bank): block-diagonal compact
// layout [i * BS + c] = M[i][(i / BS) * BS + c]
template <int Q, int BS>
struct CollC {
    double M[Q * BS], Mi[Q * BS];
};

// generated pattern-unrolled m = M f and f = M^-1 m (stream_gen.cuh, gen_stream.py)
template <int EQ, int Q, class CC>
__device__ __forceinline__ void gen_collide_mv(const CC& cc, bool inverse, const double (&x)[Q], double (&y)[Q])
{
#define GEN_MV(N)                                                                                                      \
    if (inverse)                                                                                                       \
        gen_minv_EQ##N(cc, x, y);                                                                                      \
    else                                                                                                               \
        gen_mf_EQ##N(cc, x, y);
    if constexpr (EQ == 1 && Q == 2)
    {
        GEN_MV(1)
    }
    else if constexpr (EQ == 2 && Q == 9)
    {
        GEN_MV(2)
    }
    else if constexpr (EQ == 3 && Q == 4)
    {
        GEN_MV(3)
    }
    else if constexpr (EQ == 4 && Q == 16)
    {
        GEN_MV(4)
    }
    else if constexpr (EQ == 5 && Q == 9)
    {
        GEN_MV(5)
    }
#undef GEN_MV
}

// per-population gap-1 fallback sums (stream_gen.cuh gen_fb1h_*)
template <int EQ, int Q>
__device__ __forceinline__ void gen_fb1h(int h, const double* Fin, long long cap, const double* Fj, long long capj,
                                         const int* box, const int* rim, int bstride, unsigned mask, unsigned dmask,
                                         const double* sW, double& sE, double& sA)
{
    if constexpr (EQ == 1 && Q == 2)
        gen_fb1h_EQ1(h, Fin, cap, Fj, capj, box, rim, bstride, mask, dmask, sW, sE, sA);
    else if constexpr (EQ == 2 && Q == 9)
        gen_fb1h_EQ2(h, Fin, cap, Fj, capj, box, rim, bstride, mask, dmask, sW, sE, sA);
    else if constexpr (EQ == 3 && Q == 4)
        gen_fb1h_EQ3(h, Fin, cap, Fj, capj, box, rim, bstride, mask, dmask, sW, sE, sA);
    else if constexpr (EQ == 4 && Q == 16)
        gen_fb1h_EQ4(h, Fin, cap, Fj, capj, box, rim, bstride, mask, dmask, sW, sE, sA);
    else if constexpr (EQ == 5 && Q == 9)
        gen_fb1h_EQ5(h, Fin, cap, Fj, capj, box, rim, bstride, mask, dmask, sW, sE, sA);
}

// gap-1 fallback leaf, thread per leaf (stream_gen.cuh gen_fb1t_*)
template <int EQ, int Q>
__device__ __forceinline__ void gen_fb1t(const double* Fin, long long cap, const double* Fj, long long capj,
                                         unsigned ring, int x, int y, int nx, int ny, int nxj, int nyj,
                                         int per0, int per1, unsigned mask, long long s, const double* sW, double scale,
                                         double (&f)[Q])
{
#define GEN_FB1T(N) gen_fb1t_EQ##N(Fin, cap, Fj, capj, ring, x, y, nx, ny, nxj, nyj, per0, per1, mask, s, sW, scale, f);
    if constexpr (EQ == 1 && Q == 2)
        GEN_FB1T(1)
    else if constexpr (EQ == 2 && Q == 9)
        GEN_FB1T(2)
    else if constexpr (EQ == 3 && Q == 4)
        GEN_FB1T(3)
    else if constexpr (EQ == 4 && Q == 16)
        GEN_FB1T(4)
    else if constexpr (EQ == 5 && Q == 9)
        GEN_FB1T(5)
#undef GEN_FB1T
}

template <int EQ, int Q, class RS>
__device__ __forceinline__ void gen_fb1t_rs(const double* Fin, long long cap, const double* Fj, long long capj,
                                            unsigned ring, int x, int y, int nx, int ny, int nxj, int nyj, int per0,
                                            int per1, unsigned mask, unsigned dmask, const RS& rs, long long s,
                                            const double* sW, double scale, double (&f)[Q])
{
#define GEN_FB1TR(N) gen_fb1t_rs_EQ##N(Fin, cap, Fj, capj, ring, x, y, nx, ny, nxj, nyj, per0, per1, mask, dmask, rs, s, sW, scale, f);
    if constexpr (EQ == 1 && Q == 2)
        GEN_FB1TR(1)
    else if constexpr (EQ == 2 && Q == 9)
        GEN_FB1TR(2)
    else if constexpr (EQ == 3 && Q == 4)
        GEN_FB1TR(3)
    else if constexpr (EQ == 4 && Q == 16)
        GEN_FB1TR(4)
    else if constexpr (EQ == 5 && Q == 9)
        GEN_FB1TR(5)
#undef GEN_FB1TR
}

// row i of the generated pattern-unrolled M f / M^-1 m
template <int EQ, int Q, class CC>
__device__ __forceinline__ double gen_collide_row(const CC& cc, bool inverse, int i, const double (&x)[Q])
{
#define GEN_ROW(N) return inverse ? gen_minv_row_EQ##N(cc, i, x) : gen_mf_row_EQ##N(cc, i, x);
    if constexpr (EQ == 1 && Q == 2)
    {
        GEN_ROW(1)
    }
    else if constexpr (EQ == 2 && Q == 9)
    {
        GEN_ROW(2)
    }
    else if constexpr (EQ == 3 && Q == 4)
    {
        GEN_ROW(3)
    }
    else if constexpr (EQ == 4 && Q == 16)
    {
        GEN_ROW(4)
    }
    else
    {
        GEN_ROW(5)
    }
#undef GEN_ROW
}

// Gap-1 fallback leaves (level J-1, Decision D.13b): stream AND collide, Q warps per
// block.  Blocks take chunks of the level's leaf slots (lexicographic) interleaved, so
// the resident blocks sweep the level together and the box rows they share stay in L2.
// Each block compacts the chunk's fallback leaves into a shared queue in slot order and
// processes them in batches of 32 consecutive fallback leaves:
//   A. all threads: the leaf's 5^D level-l box and the 4^D finest-level cells around its
//      children (linear indices; -1 for rim cells that are not finest leaves);
//   B. warp h, lane k: population h of leaf k -- the flattened table where exact, plus
//      the details of the rim leaves where only finer neighbours break it, or the
//      boundary rim (rim_sum) where the dependencies leave the domain;
//   C. the collision row by row: warp i computes m_i = row i of M f, warp 0 the
//      equilibrium / relaxation (and the obstacle fraction) per leaf, warp i then
//      f*_i = row i of M^-1 m' (+ blend), written to F0.
// Every value uses the same operations in the same order as K7, so the result is
// identical; the leaves' loads are spread over Q warps instead of one thread.
template <int D, int Q, int BS, int EQ, bool GEN, bool FRC = false>
__global__ void __launch_bounds__(32 * Q) k_fb1(const __grid_constant__ Geo g, const __grid_constant__ Tree tn,
                                                const __grid_constant__ Fld F0, const __grid_constant__ Fld F1,
                                                const __grid_constant__ Flags fl, const SchemeDev* scg,
                                                const __grid_constant__ Aux aux,
                                                const __grid_constant__ CollC<Q, BS> cc)
{
    constexpr int kB = D == 1 ? 5 : 25; // level-l box
    constexpr int kR = D == 1 ? 4 : 16; // finest-level 4^D box around the children
    constexpr int NT = 32 * Q;
    constexpr int kMaxE = 2 * Q * 25;
    __shared__ int sBox[kB][32];
    __shared__ int sRim[kR][32];
    __shared__ int sLin[32], sBad[32];
    __shared__ unsigned sMask[32], sDmask[32];
    __shared__ double sF[Q][32], sMo[Q][32], sAlpha[32];
    __shared__ double sW[kMaxE], sM[Q * BS], sMi[Q * BS], sS[Q], sP[8], sFeq[Q];
    __shared__ int sQ[NT + 32];
    __shared__ int sCnt[Q];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int m = g.J1 - 1, li = m - g.J0, lj = li + 1;
    if (li < 0)
        return;
    // list mode: blocks beyond the listed leaves (one 32-leaf chunk per block in the first
    // sweep) leave before the shared-memory prologue
    if (aux.fb1t && (long long)blockIdx.x * 32 >= min(aux.fb_count[3], (int)aux.fbs_cap[1]))
        return;
    {
        // gap-1 table weights in table order, scheme constants
        const int base = aux.tidx[1 * 2 * Q].x;
        const int2 last = aux.tidx[1 * 2 * Q + 2 * Q - 1];
        const int ne = min(last.x + last.y - base, kMaxE);
        for (int e = tid; e < ne; e += NT)
            sW[e] = aux.tw[base + e];
        for (int i = tid; i < Q * BS; i += NT)
        {
            sM[i] = cc.M[i];
            sMi[i] = cc.Mi[i];
        }
        for (int i = tid; i < Q; i += NT)
        {
            sS[i] = scg->s[i];
            sFeq[i] = scg->obs_feq[i];
        }
        if (tid < 8)
            sP[tid] = scg->eqp[tid];
    }
    __syncthreads();
    const int q = g.q;
    const int nL = tn.cnt[li * 4 + 0];
    const int nx = g.nx[li], ny = g.ny[li], nxj = g.nx[lj], nyj = g.ny[lj];
    const long long cap = g.cap[li], capj = g.cap[lj];
    const double scale = ldexp(1.0, D * (m - g.J1));
    // list mode (thread-per-leaf path on): the listed boundary-rim gap-1 leaves (segment 1)
    const bool from_list = aux.fb1t != 0;
    const int nfb = from_list ? min(aux.fb_count[3], (int)aux.fbs_cap[1]) : 0;
    // list mode: one batch (32 leaves) per block and chunk, so the few, long-latency
    // boundary-rim leaves spread over all blocks instead of queueing in a few
    const int CH = from_list ? 32 : NT;
    const long long nchunk = from_list ? (nfb + CH - 1) / CH : (nL + NT - 1) / NT;
    int qn = 0;
    long long ch = blockIdx.x;
    while (ch < nchunk || qn > 0)
    {
        if (ch < nchunk && qn < 32)
        {
            // append this chunk's fallback leaves to the queue, in slot order
            const long long sl = ch * NT + tid;
            int lin = -1;
            bool isfb = false;
            if (from_list)
            {
                const long long sll = ch * CH + tid;
                if (tid < CH && sll < nfb)
                {
                    lin = aux.fbs[aux.fbs_off[1] + sll];
                    isfb = true;
                }
            }
            else if (sl < nL)
            {
                lin = tn.cells[li][sl];
                isfb = (tn.skind[li][sl] & K_FB) != 0;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, isfb);
            if (lane == 0)
                sCnt[wid] = __popc(bal);
            __syncthreads();
            int off = qn, tot = qn;
            for (int w = 0; w < Q; ++w)
            {
                const int cw = sCnt[w];
                off += w < wid ? cw : 0;
                tot += cw;
            }
            if (isfb)
                sQ[off + __popc(bal & ((1u << lane) - 1u))] = lin;
            qn = tot;
            ch += gridDim.x;
            __syncthreads();
            if (qn < 32 && ch < nchunk)
                continue;
        }
        const int nb = min(qn, 32);
        // A: box and rim indices of the batch
        for (int t = tid; t < 32 * (kB + kR); t += NT)
        {
            const int k = t & 31, e = t >> 5;
            if (k >= nb)
                continue;
            int x, y;
            lin2xy_l<D>(sQ[k], ny, g.lny[li], x, y);
            if (e < kB)
            {
                const int ox = D == 1 ? e - 2 : e / 5 - 2, oy = D == 1 ? 0 : e % 5 - 2;
                int xx = x + ox, yy = y + oy;
                bool in = true;
                if (g.per0)
                    xx = mr_coord(xx, nx, 1);
                else
                    in = xx >= 0 && xx < nx;
                if (D == 2)
                {
                    if (g.per1)
                        yy = mr_coord(yy, ny, 1);
                    else
                        in = in && yy >= 0 && yy < ny;
                }
                // clamped for out-of-domain stencil cells (MR boundary rule, D.8)
                sBox[e][k] = in ? vix<D>(xx, yy, ny) : mr_vix<D>(g, m, x + ox, y + oy);
            }
            else
            {
                const int r = e - kB;
                const int rx = 2 * x - 1 + (D == 1 ? r : r / 4), ry = D == 1 ? 0 : 2 * y - 1 + r % 4;
                const bool in = (g.per0 || (rx >= 0 && rx < nxj)) && (D == 1 || g.per1 || (ry >= 0 && ry < nyj));
                const int rl = in ? mr_lin<D>(g, g.J1, rx, ry) : -1;
                sRim[r][k] = (rl >= 0 && (tn.kind[lj][rl] & K_LEAF)) ? mr_vix<D>(g, g.J1, rx, ry) : -1; // finest leaves only
            }
        }
        if (tid < nb)
        {
            const int lin = sQ[tid];
            sLin[tid] = lin;
            const int vi = vl<D>(lin, ny, g.lny[li]);
            sMask[tid] = fl.fbm[li][vi];
            sDmask[tid] = fl.fbd[li][vi];
            sBad[tid] = 0;
        }
        __syncthreads();
        // B: stream, warp = population
        if (lane < nb && wid < Q)
        {
            const int h = wid, k = lane;
            const int lin = sLin[k];
            const unsigned mask = sMask[k], dmask = sDmask[k];
            double sum[2] = {0.0, 0.0};
            if constexpr (GEN)
                gen_fb1h<EQ, Q>(h, F1.f[li], cap, F1.f[lj], capj, &sBox[0][k], &sRim[0][k], 32, mask, dmask, sW, sum[0],
                                sum[1]);
            else
            {
                const double* Fh = F1.f[li] + (long long)h * cap;
                const double* Fj = F1.f[lj] + (long long)h * capj;
                const int ex = scg->eta[h][0], ey = D == 1 ? 0 : scg->eta[h][1];
                int x, y;
                lin2xy_l<D>(lin, ny, g.lny[li], x, y);
                for (int side = 0; side < 2; ++side)
                {
                    const int pair = 2 * h + side;
                    if ((dmask >> pair) & 1u)
                        continue;
                    double acc = 0.0;
                    const int2 ti = aux.tidx[(1 * q + h) * 2 + side];
                    for (int e = ti.x; e < ti.x + ti.y; ++e)
                    {
                        const int2 o = aux.toff[e];
                        const int bb = D == 1 ? o.x + 2 : (o.x + 2) * 5 + (o.y + 2);
                        acc = __dadd_rn(acc, __dmul_rn(aux.tw[e], Fh[sBox[bb][k]]));
                    }
                    if ((mask >> pair) & 1u)
                    {
                        // Decision D.13b: + details of the rim cells that are finest leaves
                        for (int r = 0; r < kR; ++r)
                        {
                            const int dx = D == 1 ? r : r / 4, dy = D == 1 ? 0 : r % 4;
                            const int xr = 2 * x - 1 + dx, yr = D == 1 ? 0 : 2 * y - 1 + dy;
                            const bool inb = dx >= 1 && dx <= 2 && (D == 1 || (dy >= 1 && dy <= 2));
                            const bool ine = (dx + ex) >= 1 && (dx + ex) <= 2 &&
                                             (D == 1 || ((dy + ey) >= 1 && (dy + ey) <= 2));
                            if (!(side == 0 ? (ine && !inb) : (inb && !ine)))
                                continue;
                            const int sj = sRim[r][k];
                            if (sj < 0)
                                continue;
                            const int xc = mr_coord(xr, nxj, g.per0), yc = D == 2 ? mr_coord(yr, nyj, g.per1) : 0;
                            const int pdx = (dx + 1) / 2 - 1, pdy = D == 1 ? 0 : (dy + 1) / 2 - 1;
                            constexpr int NS = D == 1 ? 3 : 9;
                            double sv[NS];
                            for (int o = 0; o < NS; ++o)
                            {
                                const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
                                const int bb = D == 1 ? pdx + ox + 2 : (pdx + ox + 2) * 5 + (pdy + oy + 2);
                                sv[o] = Fh[sBox[bb][k]];
                            }
                            acc = __dadd_rn(acc, __dsub_rn(Fj[sj], mr_predict<D>(sv, xc & 1, yc & 1)));
                        }
                    }
                    sum[side] = acc;
                }
            }
            if (dmask)
            {
                int x, y;
                lin2xy_l<D>(lin, ny, g.lny[li], x, y);
                for (int side = 0; side < 2; ++side)
                    if ((dmask >> (2 * h + side)) & 1u)
                    {
                        const int bx0 = 2 * x, bx1 = bx0 + 2, by0 = D == 1 ? 0 : 2 * y, by1 = D == 1 ? 1 : by0 + 2;
                        sum[side] = rim_sum<D>(g, tn, F1, scg, h, side, bx0, bx1, by0, by1, li, lin, aux);
                    }
            }
            sF[h][k] = __dadd_rn(F1.f[li][(long long)h * cap + vl<D>(lin, ny, g.lny[li])], __dmul_rn(scale, __dsub_rn(sum[0], sum[1])));
        }
        __syncthreads();
        // C1: m_i = row i of M f
        if (lane < nb && wid < Q)
        {
            const int i = wid, k = lane;
            double f[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j)
                f[j] = sF[j][k];
            double acc = 0.0;
            if constexpr (GEN)
                acc = gen_collide_row<EQ, Q>(cc, false, i, f);
            else
            {
                const int b0 = (i / BS) * BS;
#pragma unroll
                for (int j = 0; j < BS; ++j)
                    acc = __dadd_rn(acc, __dmul_rn(sM[i * BS + j], f[b0 + j]));
            }
            sMo[i][k] = acc;
        }
        __syncthreads();
        // C2: equilibrium and relaxation per leaf; obstacle fraction
        if (wid == 0 && lane < nb)
        {
            const int k = lane;
            double mo[Q], meq[Q];
#pragma unroll
            for (int i = 0; i < Q; ++i)
                mo[i] = sMo[i][k];
            equilibrium_t<EQ, Q>(sP, scg->lambda, mo, meq);
#pragma unroll
            for (int i = 0; i < Q; ++i)
                sMo[i][k] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, sS[i]), mo[i]), __dmul_rn(sS[i], meq[i]));
            double alpha = 0.0;
            if constexpr (EQ == MRLBM_EQ_NS_D2Q9 && D == 2)
            {
                if (scg->obstacle == 1)
                {
                    int x, y;
                    lin2xy_l<D>(sLin[k], ny, g.lny[li], x, y);
                    alpha = obstacle_alpha_cached(aux, li, x, y);
                    if constexpr (FRC)
                        if (alpha > 0.0)
                            force_store(aux, g, scg, m, x, y, alpha, sMo[1][k], sMo[2][k]);
                }
            }
            sAlpha[k] = alpha;
        }
        __syncthreads();
        // C3: f*_i = row i of M^-1 m', blend, store
        if (lane < nb && wid < Q)
        {
            const int i = wid, k = lane;
            double mo[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j)
                mo[j] = sMo[j][k];
            double fi = 0.0;
            if constexpr (GEN)
                fi = gen_collide_row<EQ, Q>(cc, true, i, mo);
            else
            {
                const int b0 = (i / BS) * BS;
#pragma unroll
                for (int j = 0; j < BS; ++j)
                    fi = __dadd_rn(fi, __dmul_rn(sMi[i * BS + j], mo[b0 + j]));
            }
            const double alpha = sAlpha[k];
            if (alpha > 0.0)
                fi = __dadd_rn(__dmul_rn(alpha, sFeq[i]), __dmul_rn(__dsub_rn(1.0, alpha), fi));
            if (!isfinite(fi))
                sBad[k] = 1;
            F0.f[li][(long long)i * cap + vl<D>(sLin[k], ny, g.lny[li])] = fi;
        }
        // shift the queue
        const int rest = qn - nb;
        const int carry = tid < rest ? sQ[32 + tid] : 0;
        __syncthreads();
        if (tid < rest)
            sQ[tid] = carry;
        if (tid < nb && sBad[tid])
            flag_err(aux.err, 1);
        qn = rest;
        __syncthreads();
    }
}

// K7: table-path stream + collision +
// obstacle blend, one thread per leaf.  Fallback leaves take their post-stream
// populations from K8 (already in F0).  BS = block size of the block-diagonal M.
// MODE 0 streams the table-path leaves only (no calls, no stack: the hot kernel);
// MODE 1 the fallback leaves at gap 0 (boundary rim) and gap >= 2 (values from K8).
template <int D, int Q, int BS, int EQ, bool GEN, int MODE, int GC, bool FRC = false>
__global__ void __launch_bounds__(256, GC == 1 ? 2 : 3)
    k_stream_collide(const __grid_constant__ Geo g, const __grid_constant__ Tree tn, const __grid_constant__ Fld F0,
                     const __grid_constant__ Fld F1, const __grid_constant__ Flags fl, const SchemeDev* scg,
                     const __grid_constant__ LGrid lg_, const __grid_constant__ Aux aux,
                     const __grid_constant__ CollC<Q, BS> cc)
{
    LSETUP;
    constexpr int kMaxE = 2 * Q * 25;
    constexpr int kU = D == 1 ? 5 : 25; // distinct table offsets at one gap (5^D box)
    constexpr int kT = 256;
    __shared__ double sM[Q * BS], sMi[Q * BS], sS[Q], sP[8], sW[kMaxE];
    __shared__ uint8_t sU[kMaxE];        // entry -> index into the distinct offsets
    __shared__ int2 sIdx[2 * Q];
    __shared__ int2 sUoff[kU];
    __shared__ int sNU;
    __shared__ int sSlot[kU][kT];        // per-thread neighbour slots
    __shared__ double sFeq[Q];
    __shared__ int2 sEta[Q];
    const int gap = g.J1 - m;
    for (int i = threadIdx.x; i < Q * BS; i += blockDim.x)
    {
        const int r = i / BS, c = i % BS;
        const int col = (r / BS) * BS + c;
        sM[i] = scg->M[r * Q + col];
        sMi[i] = scg->Minv[r * Q + col];
    }
    for (int i = threadIdx.x; i < Q; i += blockDim.x)
    {
        sS[i] = scg->s[i];
        sFeq[i] = scg->obs_feq[i];
        sEta[i] = make_int2(scg->eta[i][0], scg->eta[i][1]);
    }
    if (threadIdx.x < 8)
        sP[threadIdx.x] = scg->eqp[threadIdx.x];
    // this gap's flattened tables and distinct offsets (deduplicated on the host)
    {
        const int2 gu = aux.guidx[gap];
        const int base = aux.tidx[gap * 2 * Q].x;
        const int2 last = aux.tidx[gap * 2 * Q + 2 * Q - 1];
        const int ne = min(last.x + last.y - base, kMaxE);
        for (int t = threadIdx.x; t < 2 * Q; t += blockDim.x)
        {
            const int2 ti = aux.tidx[gap * 2 * Q + t];
            sIdx[t] = make_int2(ti.x - base, ti.y);
        }
        for (int e = threadIdx.x; e < ne; e += blockDim.x)
        {
            sU[e] = aux.tu[base + e];
            sW[e] = aux.tw[base + e];
        }
        for (int u = threadIdx.x; u < gu.y && u < kU; u += blockDim.x)
            sUoff[u] = aux.guoff[gu.x + u];
        if (threadIdx.x == 0)
            sNU = min(gu.y, kU);
    }
    __syncthreads();
    const int nu = sNU;
    const int li = m - g.J0;
    const int nL = tn.cnt[li * 4 + 0];
    const int nx = g.nx[li], ny = g.ny[li];
    const long long cap = g.cap[li];
    const double scale = ldexp(1.0, D * (m - g.J1));
    const double* Fin = F1.f[li];
    double* Fout = F0.f[li];
    const int per0 = g.per0, per1 = g.per1;
    int* myslot = &sSlot[0][threadIdx.x];
    // grid-stride over the leaf slots with the next slot's (index, kind) loaded one
    // iteration ahead, so the value gathers never wait on the slot list
    // MODE 3 / 5 take their leaves from the fallback segment lists instead of the slots
    const int* lst = nullptr;
    int nItems = nL;
    if constexpr (MODE == 2 || MODE == 3 || MODE == 5)
    {
        constexpr int seg = MODE == 5 ? 0 : (MODE == 3 ? 1 : 2);
        lst = aux.fbs + aux.fbs_off[seg];
        nItems = min(aux.fb_count[2 + seg], (int)aux.fbs_cap[seg]);
    }
    const long long sstep = (long long)lvg_ * blockDim.x;
    long long s = (long long)lvb_ * blockDim.x + threadIdx.x;
    int lin_next = s < nItems ? (lst ? lst[s] : tn.cells[li][s]) : 0;
    uint8_t kd_next = s < nItems ? (lst ? (uint8_t)(K_LEAF | K_FB) : tn.skind[li][s]) : 0;
    for (; s < nItems; s += sstep)
    {
        const int lin = lin_next;
        const int vself = vl<D>(lin, ny, g.lny[li]);
        const uint8_t kd = kd_next;
        if (s + sstep < nItems)
        {
            lin_next = lst ? lst[s + sstep] : tn.cells[li][s + sstep];
            kd_next = lst ? (uint8_t)(K_LEAF | K_FB) : tn.skind[li][s + sstep];
        }
        if (((kd & K_FB) != 0) != (MODE >= 1))
            continue;
        constexpr bool fb = MODE == 1 || MODE == 5;
        if (fb && gap == 1)
            continue; // streamed and collided by k_fb1 / MODE 2
        double f[Q];
        if constexpr (MODE == 2 || MODE == 3)
        {
            // gap-1 fallback leaf, one thread per leaf: table + details of the finest-leaf
            // rim cells (Decision D.13b), the same operands and order as k_fb1.  MODE 2: the
            // leaves without domain-leaving pairs (slot scan); MODE 3: the listed others,
            // whose domain-leaving pairs take the boundary rim sum (rim_sum)
            if (MODE == 2 && fl.fbd[li][vself] != 0)
                continue;
            int x, y;
            lin2xy_l<D>(lin, ny, g.lny[li], x, y);
            // finest leaves among the 4^D cells around the children (the E-rim ring;
            // the inner 2^D are the leaf's own children, never leaves): one bit each
            const int nxj = g.nx[li + 1], nyj = g.ny[li + 1];
            const uint8_t* kj = tn.kind[li + 1];
            unsigned ring = 0;
#pragma unroll
            for (int r = 0; r < (D == 1 ? 4 : 16); ++r)
            {
                const int dx = D == 1 ? r : r >> 2, dy = D == 1 ? 0 : r & 3;
                if (dx >= 1 && dx <= 2 && (D == 1 || (dy >= 1 && dy <= 2)))
                    continue;
                int xr = 2 * x - 1 + dx, yr = D == 1 ? 0 : 2 * y - 1 + dy;
                if (xr < 0 || xr >= nxj)
                {
                    if (!per0)
                        continue;
                    xr = mr_coord(xr, nxj, 1);
                }
                if (D == 2 && (yr < 0 || yr >= nyj))
                {
                    if (!per1)
                        continue;
                    yr = mr_coord(yr, nyj, 1);
                }
                if (kj[xy2lin<D>(xr, yr, nyj)] & K_LEAF)
                    ring |= 1u << r;
            }
            if constexpr (MODE == 2)
                gen_fb1t<EQ, Q>(Fin, cap, F1.f[li + 1], g.cap[li + 1], ring, x, y, nx, ny, nxj, nyj, per0, per1,
                                fl.fbm[li][vself], vself, sW, scale, f);
            else
            {
                const RimCold<D> rs{&g, &tn, &F1, scg, &aux, x, y, li, lin};
                gen_fb1t_rs<EQ, Q>(Fin, cap, F1.f[li + 1], g.cap[li + 1], ring, x, y, nx, ny, nxj, nyj, per0, per1,
                                   fl.fbm[li][vself], fl.fbd[li][vself], rs, vself, sW, scale, f);
            }
        }
        else if (fb && gap >= kDeepGap)
        {
            // deep-gap fallback leaf: post-stream populations from K8
#pragma unroll
            for (int h = 0; h < Q; ++h)
                f[h] = Fout[(long long)h * cap + vself];
        }
        else if (GEN && !fb)
        {
            int x, y;
            lin2xy_l<D>(lin, ny, g.lny[li], x, y);
            gen_stream<EQ, Q, GC>(gap, Fin, cap, x, y, nx, ny, per0, per1, vself, sW, scale, f);
        }
        else
        {
            int x, y;
            lin2xy_l<D>(lin, ny, g.lny[li], x, y);
            // all neighbour slots first (independent loads), then pure gathers
            for (int u = 0; u < nu; ++u)
            {
                const int2 o = sUoff[u];
                int xx = x + o.x, yy = y + o.y;
                bool in = true;
                if (per0)
                    xx = mr_coord(xx, nx, 1);
                else
                    in = xx >= 0 && xx < nx;
                if (D == 2)
                {
                    if (per1)
                        yy = mr_coord(yy, ny, 1);
                    else
                        in = in && yy >= 0 && yy < ny;
                }
                myslot[u * kT] = in ? vix<D>(xx, yy, ny) : -1;
            }
            const unsigned mask = fb ? fl.fbm[li][vself] : 0u;
            if (mask)
            {
                // shallow fallback leaf: table where exact, recursive rim elsewhere
                const int side_n = 1 << gap;
                const int bx0 = x * side_n, bx1 = bx0 + side_n;
                const int by0 = D == 1 ? 0 : y * side_n, by1 = D == 1 ? 1 : by0 + side_n;
                for (int h = 0; h < Q; ++h)
                {
                    const double* Fh = Fin + (long long)h * cap;
                    double sum[2];
                    for (int side = 0; side < 2; ++side)
                    {
                        double acc = 0.0;
                        if ((mask >> (2 * h + side)) & 1u)
                            acc = rim_sum<D>(g, tn, F1, scg, h, side, bx0, bx1, by0, by1, li, lin, aux);
                        else
                        {
                            const int2 ti = sIdx[2 * h + side];
                            for (int e = ti.x; e < ti.x + ti.y; ++e)
                            {
                                const int sl = myslot[sU[e] * kT];
                                const double v = sl >= 0 ? Fh[sl] : 0.0;
                                acc = __dadd_rn(acc, __dmul_rn(sW[e], v));
                            }
                        }
                        sum[side] = acc;
                    }
                    f[h] = __dadd_rn(Fh[vself], __dmul_rn(scale, __dsub_rn(sum[0], sum[1])));
                }
            }
            else if (gap == 0)
            {
                // finest level: every table has at most one entry (E = {-eta}, A = {0});
                // branch-free so all 2Q gathers are independent and in flight together
                double vE[Q], vA[Q], fs[Q];
#pragma unroll
                for (int h = 0; h < Q; ++h)
                {
                    const double* Fh = Fin + (long long)h * cap;
                    const int2 tE = sIdx[2 * h], tA = sIdx[2 * h + 1];
                    const int slE = tE.y ? myslot[sU[tE.x] * kT] : -1;
                    const int slA = tA.y ? myslot[sU[tA.x] * kT] : -1;
                    fs[h] = Fh[vself];
                    vE[h] = slE >= 0 ? Fh[slE] : 0.0;
                    vA[h] = slA >= 0 ? Fh[slA] : 0.0;
                }
#pragma unroll
                for (int h = 0; h < Q; ++h)
                {
                    const int2 tE = sIdx[2 * h], tA = sIdx[2 * h + 1];
                    const double sE = tE.y ? __dadd_rn(0.0, __dmul_rn(sW[tE.x], vE[h])) : 0.0;
                    const double sA = tA.y ? __dadd_rn(0.0, __dmul_rn(sW[tA.x], vA[h])) : 0.0;
                    f[h] = __dadd_rn(fs[h], __dmul_rn(scale, __dsub_rn(sE, sA)));
                }
            }
            else
            {
#pragma unroll
                for (int h = 0; h < Q; ++h)
                {
                    const double* Fh = Fin + (long long)h * cap;
                    const double fs = Fh[vself];
                    double sum[2];
#pragma unroll
                    for (int side = 0; side < 2; ++side)
                    {
                        const int2 ti = sIdx[2 * h + side];
                        double acc = 0.0;
#pragma unroll 8
                        for (int e = ti.x; e < ti.x + ti.y; ++e)
                        {
                            const int sl = myslot[sU[e] * kT];
                            const double v = sl >= 0 ? Fh[sl] : 0.0;
                            acc = __dadd_rn(acc, __dmul_rn(sW[e], v));
                        }
                        sum[side] = acc;
                    }
                    f[h] = __dadd_rn(fs, __dmul_rn(scale, __dsub_rn(sum[0], sum[1])));
                }
            }
        }
        // collide: m = M f (block diagonal, DenseMatrix::multiply order),
        // m' = (1-s) m + s m^eq, f* = M^-1 m'
        double mo[Q], meq[Q];
        if constexpr (GEN)
            gen_collide_mv<EQ, Q>(cc, false, f, mo);
        else
        {
#pragma unroll
            for (int i = 0; i < Q; ++i)
            {
                const int b0 = (i / BS) * BS;
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < BS; ++j)
                    acc = __dadd_rn(acc, __dmul_rn(sM[i * BS + j], f[b0 + j]));
                mo[i] = acc;
            }
        }
        equilibrium_t<EQ, Q>(sP, scg->lambda, mo, meq);
#pragma unroll
        for (int i = 0; i < Q; ++i)
            mo[i] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, sS[i]), mo[i]), __dmul_rn(sS[i], meq[i]));
        if constexpr (GEN)
            gen_collide_mv<EQ, Q>(cc, true, mo, f);
        else
        {
#pragma unroll
            for (int i = 0; i < Q; ++i)
            {
                const int b0 = (i / BS) * BS;
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < BS; ++j)
                    acc = __dadd_rn(acc, __dmul_rn(sMi[i * BS + j], mo[b0 + j]));
                f[i] = acc;
            }
        }
        if constexpr (EQ == MRLBM_EQ_NS_D2Q9 && D == 2)
        {
            if (scg->obstacle == 1)
            {
                int x, y;
                lin2xy_l<D>(lin, ny, g.lny[li], x, y);
                const double alpha = obstacle_alpha_cached(aux, li, x, y);
                if (alpha > 0.0)
                {
                    if constexpr (FRC)
                        force_store(aux, g, scg, m, x, y, alpha, mo[1], mo[2]);
#pragma unroll
                    for (int h = 0; h < Q; ++h)
                        f[h] = __dadd_rn(__dmul_rn(alpha, sFeq[h]), __dmul_rn(__dsub_rn(1.0, alpha), f[h]));
                }
            }
        }
        bool bad = false;
#pragma unroll
        for (int h = 0; h < Q; ++h)
        {
            bad = bad || !isfinite(f[h]);
            Fout[(long long)h * cap + vself] = f[h];
        }
        if (bad)
            flag_err(aux.err, 1);
    }
}

__global__ void k_count_updates(const int* cnt, int nlev, long long* acc, int* step_no)
{
    if (threadIdx.x == 0 && blockIdx.x == 0)
    {
        long long s = 0;
        for (int i = 0; i < nlev; ++i)
            s += cnt[i * 4];
        *acc += s;
        *step_no += 1;
    }
}

// loading: mark loaded leaves and their ancestors; scatter values after compaction
template <int D>
__global__ void k_load_mark(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, const int* lins, int n, int m)
{
    const int li = m - g.J0;
    const int ny = g.ny[li];
    GRID_STRIDE(i, 0, n)
    {
        const int lin = lins[i];
        fl.keep[li][lin] = 1; // loaded-leaf marker
        if (m > g.J0)
        {
            int x, y;
            lin2xy_l<D>(lin, ny, g.lny[li], x, y);
            fl.rn[li - 1][xy2lin<D>(x >> 1, y >> 1, g.ny[li - 1])] = 1;
        }
    }
}

template <int D>
__global__ void k_closure_dense(const __grid_constant__ Geo g, const __grid_constant__ Flags fl, int m)
{
    const int li = m - g.J0;
    const int ny = g.ny[li];
    const long long n = (long long)g.nx[li] * ny;
    GRID_STRIDE(i, 0, n)
    {
        if (!fl.rn[li][i])
            continue;
        int x, y;
        lin2xy_l<D>((int)i, ny, g.lny[li], x, y);
        fl.rn[li - 1][xy2lin<D>(x >> 1, y >> 1, g.ny[li - 1])] = 1;
    }
}

// load: coordinates (n x d) -> linear indices, with a domain check
__global__ void k_idx_to_lin(const int32_t* idx, int n, int d, int nx, int ny, int32_t* lin, int* bad)
{
    GRID_STRIDE(i, 0, n)
    {
        const int x = idx[i * d], y = d == 2 ? idx[i * d + 1] : 0;
        if (x < 0 || x >= nx || y < 0 || y >= ny)
        {
            atomicAdd(bad, 1);
            lin[i] = 0;
            continue;
        }
        lin[i] = d == 2 ? x * ny + y : x;
    }
}

// read: linear indices -> coordinates
__global__ void k_lin_to_idx(const int32_t* lin, int n, int d, int ny, int32_t* idx)
{
    GRID_STRIDE(i, 0, n)
    {
        const int l = lin[i];
        if (d == 2)
        {
            idx[2 * i] = l / ny;
            idx[2 * i + 1] = l - (l / ny) * ny;
        }
        else
            idx[i] = l;
    }
}

__global__ void k_load_scatter(const int* lins, const double* fin, int n, int q, const uint8_t* kind, double* F,
                               long long cap, int* err, int d, int ny, int lny)
{
    GRID_STRIDE(i, 0, n)
    {
        const int lin = lins[i];
        if (kind[lin] != K_LEAF)
        {
            atomicAdd(&err[2], 1);
            continue;
        }
        const int vi = d == 2 ? vl<2>(lin, ny, lny) : lin;
        for (int h = 0; h < q; ++h)
            F[(long long)h * cap + vi] = fin[(long long)h * n + i];
    }
}

// read: gather the leaves (slot order) of a level into packed SoA q x n
__global__ void k_gather_leaves(const int32_t* cells, int n, int q, const double* F, long long cap, double* out, int d,
                                int ny, int lny)
{
    GRID_STRIDE(i, 0, n)
    {
        const int lin = cells[i];
        const int vi = d == 2 ? vl<2>(lin, ny, lny) : lin;
        for (int h = 0; h < q; ++h)
            out[(long long)h * n + i] = F[(long long)h * cap + vi];
    }
}

// ---------------------------------------------------------------- diagnostics
// Internal values of the current tree = projection of its leaves (the values K1 of the
// next step recomputes identically), runtime q.  Slots [nL, nL + nI) of level m.
template <int D>
__global__ void k_recon_project(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Fld F, int m, int q)
{
    const int li = m - g.J0;
    const int nL = t.cnt[li * 4 + 0], nI = t.cnt[li * 4 + 1];
    const int ny = g.ny[li], ny1 = g.ny[li + 1];
    const long long cap = g.cap[li], cap1 = g.cap[li + 1];
    GRID_STRIDE(s, nL, nL + nI)
    {
        const int plin = t.cells[li][s];
        int px, py;
        lin2xy<D>(plin, ny, px, py);
        for (int h = 0; h < q; ++h)
        {
            const double* src = F.f[li + 1] + (long long)h * cap1;
            double acc = 0.0;
            for (int c = 0; c < (1 << D); ++c)
            {
                const int dx = D == 1 ? c : (c >> 1), dy = D == 1 ? 0 : (c & 1);
                acc = __dadd_rn(acc, src[vix<D>(2 * px + dx, 2 * py + dy, ny1)]);
            }
            F.f[li][(long long)h * cap + vix<D>(px, py, ny)] = __ddiv_rn(acc, (double)(1 << D));
        }
    }
}

// Zero-detail reconstruction f^^ of every cell of level m: the
// complete-tree value where the cell is in R(Lambda), else the prediction from the
// (complete) reconstruction of level m-1 with the clamp / wrap stencil rule (D.8).
// Level J0 lies entirely in R.  Same recursion as the oracle's rec().
template <int D>
__global__ void k_recon_level(const __grid_constant__ Geo g, const __grid_constant__ Tree t, const __grid_constant__ Fld S, const __grid_constant__ Fld R, int m, int q)
{
    const int li = m - g.J0;
    const long long cap = g.cap[li];
    const int ny = g.ny[li];
    GRID_STRIDE(i, 0, cap)
    {
        const int lin = (int)i;
        if (t.kind[li][lin] & (K_LEAF | K_INT))
        {
            // R is row-major (lexicographic output), S in sibling blocks
            const int vi = vl<D>(lin, ny, g.lny[li]);
            for (int h = 0; h < q; ++h)
                R.f[li][(long long)h * cap + lin] = S.f[li][(long long)h * cap + vi];
            continue;
        }
        int x, y;
        lin2xy<D>(lin, ny, x, y);
        const int px = x >> 1, py = D == 1 ? 0 : (y >> 1);
        int st[D == 1 ? 3 : 9];
        for (int o = 0; o < (D == 1 ? 3 : 9); ++o)
        {
            const int ox = D == 1 ? o - 1 : o / 3 - 1, oy = D == 1 ? 0 : o % 3 - 1;
            st[o] = mr_lin<D>(g, m - 1, px + ox, py + oy);
        }
        const long long capp = g.cap[li - 1];
        for (int h = 0; h < q; ++h)
        {
            const double* P = R.f[li - 1] + (long long)h * capp;
            double sv[D == 1 ? 3 : 9];
            for (int o = 0; o < (D == 1 ? 3 : 9); ++o)
                sv[o] = P[st[o]];
            R.f[li][(long long)h * cap + lin] = mr_predict<D>(sv, x & 1, D == 1 ? 0 : (y & 1));
        }
    }
}

// E[m] partial sums: per block, sum |m_a - m_b| and sum |m_b| with
// m = sum_h row[h] f^h (h ascending); fixed thread -> cell map and a fixed tree
// reduction, so the result is deterministic for a given grid.
__global__ void __launch_bounds__(256) k_moment_err(const double* A, const double* B, long long cap, int q,
                                                    const double* row, long long n, double* part)
{
    __shared__ double s0[256], s1[256];
    double e = 0.0, r = 0.0;
    GRID_STRIDE(i, 0, n)
    {
        double ma = 0.0, mb = 0.0;
        for (int h = 0; h < q; ++h)
        {
            ma = __dadd_rn(ma, __dmul_rn(row[h], A[(long long)h * cap + i]));
            mb = __dadd_rn(mb, __dmul_rn(row[h], B[(long long)h * cap + i]));
        }
        e = __dadd_rn(e, fabs(__dsub_rn(ma, mb)));
        r = __dadd_rn(r, fabs(mb));
    }
    s0[threadIdx.x] = e;
    s1[threadIdx.x] = r;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1)
    {
        if ((int)threadIdx.x < w)
        {
            s0[threadIdx.x] = __dadd_rn(s0[threadIdx.x], s0[threadIdx.x + w]);
            s1[threadIdx.x] = __dadd_rn(s1[threadIdx.x], s1[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
    {
        part[2 * blockIdx.x] = s0[0];
        part[2 * blockIdx.x + 1] = s1[0];
    }
}

} // namespace mrlbm_b200

using namespace mrlbm_b200;

// ====================================================================== host context
struct mrlbm_ctx {
    mrlbm_b200::Engine3D* e3 = nullptr; // scheme.d == 3: the 3D engine (mrlbm_step3d.cu) owns everything
    mrlbm_scheme_spec sc{};
    mrlbm_run_config rc{};
    int D = 0, q = 0, J0 = 0, J1 = 0, nlev = 0;
    Geo geo{};
    cudaStream_t stream = nullptr;
    int32_t* cells[2][kL]{};
    uint8_t* skind[2][kL]{}; // per tree version: kinds in slot order
    uint8_t* kind2[2][kL]{}; // per tree version: dense cell kinds
    int* cnt[2]{};
    uint8_t* rn[kL]{};
    uint8_t* keep[kL]{};
    uint8_t** dirty_d = nullptr; // device array of keep[] pointers (K6 dirty flags; keep is free after K4)
    unsigned* fbmd[kL]{};
    unsigned* fbdd[kL]{};
    double* F[2][kL]{};
    int* tiles[kL]{};
    long long ntiles[kL]{};
    SchemeDev* sch = nullptr;
    int* err = nullptr;
    int* fbc = nullptr;
    int* fbs = nullptr; // fallback segment lists (Aux::fbs)
    long long fbs_off[3]{}, fbs_cap[3]{};
    int2* fbl = nullptr;
    unsigned* fbm = nullptr;
    unsigned* fbdm = nullptr;
    long long fbcap = 0;
    long long* upd = nullptr;
    int2* tidx = nullptr;
    int2* toff = nullptr;
    double* tw = nullptr;
    int4* tdep = nullptr;
    int2* tpidx = nullptr;
    int2* tpar = nullptr;
    int4* udep = nullptr;
    int2* guidx = nullptr;
    int2* guoff = nullptr;
    uint8_t* tu = nullptr;
    int2* upidx = nullptr;
    int2* upar = nullptr;
    int2* etad = nullptr;
    unsigned short* pmaskd = nullptr;
    unsigned short* umaskd = nullptr;
    int cur = 0;
    int curf = 0; // F[curf] holds the state f* (dense, indexed by the linear cell index)
    bool committed = false;
    int profiling = 0; // 1: an event after every kernel, one stream; 2: phase events only, forks active
    bool use_graph = true;
    bool use_gen = false; // generated stream / collision path (built-in velocity sets)
    bool use_fb1t = true; // gap-1 fallback leaves thread per leaf (K7 MODE 2) instead of k_fb1; MRLBM_NO_FB1T=1 turns it off
    bool rim_tpl = false; // boundary-rim gap-1 leaves thread per leaf too (K7 MODE 3, MRLBM_RIM_TPL=1) instead of k_fb1 (list)
    // K1+K2 fused per level (MRLBM_FUSE_PD=1): measured slower than the separate
    // kernels (re-projecting the internal stencil neighbours costs more than the
    // second read of the children), so off by default
    bool fuse_pd = false;
    // K8 one warp per (leaf, population) (MRLBM_K8_WARP=1, round-1 kernel) instead of one thread
    bool k8_warp = false;
    // K8 one block per 32-leaf chunk with shared box indices (MRLBM_K8_BLOCK=1): measured slower,
    // 1.59 vs 1.09 ms per window step (the block waits at every chunk for its longest rim)
    bool k8_block = false;
    // the stream + collide launches are independent of one another (disjoint leaves, all read the
    // transferred state) except K8 -> MODE 1; they fork onto side streams inside the step graph so
    // that the small latency-bound ones overlap (MRLBM_SERIAL_STREAM=1: one stream)
    bool fork_stream = true;
    cudaStream_t side[5]{};
    cudaEvent_t ev_fork = nullptr, ev_join[5]{};
    // long-rim leaves (gap >= kLongGap) in the warp-cooperative K8 launch (MRLBM_K8_LONG_GAP=g sets the
    // threshold, 0 keeps all deep-gap leaves in the thread kernel)
    int k8_long = kLongGap;
    int k8_occ = 4; // K8 thread kernel: resident blocks per SM the register budget is set for (MRLBM_K8_OCC)
    bool gen_ok = false;  // the generated code's constants match this scheme
    unsigned emask = 0;   // H(a): parent offsets (3^d bits) of the eta-shifted children
    cudaGraphExec_t graph[2]{};
    // load staging (device): per level, coordinates -> linear indices; the values are
    // staged in F[1] (free until the first step)
    int32_t* ld_idx[kL]{};
    int32_t* ld_lin[kL]{};
    long long ld_n[kL]{};
    int* ld_bad = nullptr;
    // obstacle force tracking (mrlbm_set_force_tracking)
    double* frc = nullptr;
    double* alpha_tab = nullptr; // obstacle alpha per cell of the boxes (Aux::alpha_tab)
    long long frc_n = 0; // cells over all level boxes
    long long frc_off[kL]{};
    int frc_x0[kL]{}, frc_y0[kL]{}, frc_nx[kL]{}, frc_ny[kL]{};
    double* fhist = nullptr;
    int* fhn = nullptr;
    int* rdcnt = nullptr; // read-back: level totals of the lexicographic re-sort
    // near-threshold tie log (mrlbm_tie_log)
    mrlbm_tie_record* ties = nullptr;
    int* tie_n = nullptr;
    int* step_no = nullptr;
    int tie_cap = 1 << 16;
    int fcap = 0;
    cudaEvent_t ev[16]{};
    double phase_ms[MRLBM_PHASE_COUNT]{};
    std::string err_msg;
    int grid_cap = 148 * 8;
    long long kernels_per_step = 0; // counted while enqueueing one step
    long long kcount = 0;
    // per-launch timing (profiling mode only): event after every kernel
    std::vector<cudaEvent_t> kev;
    std::vector<std::pair<std::string, int>> klabel;
    std::map<std::pair<std::string, int>, std::pair<double, int>> kacc;
    int kn = 0;
};

namespace {

int set_err(mrlbm_ctx* c, int code, const std::string& msg)
{
    if (c)
        c->err_msg = msg;
    return code;
}

#define CU(call)                                                                                                       \
    do                                                                                                                 \
    {                                                                                                                  \
        cudaError_t e_ = (call);                                                                                       \
        if (e_ != cudaSuccess)                                                                                         \
            return set_err(ctx, MRLBM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));                \
    } while (0)

Tree tree_of(mrlbm_ctx* c, int v)
{
    Tree t{};
    for (int i = 0; i < c->nlev; ++i)
    {
        t.kind[i] = c->kind2[v][i];
        t.cells[i] = c->cells[v][i];
        t.skind[i] = c->skind[v][i];
    }
    t.cnt = c->cnt[v];
    return t;
}

Fld fld_of(mrlbm_ctx* c, int v)
{
    Fld f{};
    for (int i = 0; i < c->nlev; ++i)
        f.f[i] = c->F[v][i];
    return f;
}

Flags flags_of(mrlbm_ctx* c, int v)
{
    Flags f{};
    for (int i = 0; i < c->nlev; ++i)
    {
        f.kind[i] = c->kind2[v][i];
        f.rn[i] = c->rn[i];
        f.keep[i] = c->keep[i];
        f.fbm[i] = c->fbmd[i];
        f.fbd[i] = c->fbdd[i];
    }
    return f;
}

Aux aux_of(mrlbm_ctx* c)
{
    Aux a{};
    a.err = c->err;
    a.fb_count = c->fbc;
    a.fb_list = c->fbl;
    a.fb_mask = c->fbm;
    a.fb_dmask = c->fbdm;
    a.fb_cap = c->fbcap;
    a.updates = c->upd;
    a.tidx = c->tidx;
    a.toff = c->toff;
    a.tw = c->tw;
    a.tdep = c->tdep;
    a.tpidx = c->tpidx;
    a.tpar = c->tpar;
    a.udep = c->udep;
    a.guidx = c->guidx;
    a.guoff = c->guoff;
    a.tu = c->tu;
    a.upidx = c->upidx;
    a.upar = c->upar;
    a.eta = c->etad;
    a.pmask = c->pmaskd;
    a.umask = c->umaskd;
    a.frc = c->frc;
    a.alpha_tab = c->alpha_tab;
    a.ties = c->ties;
    a.tie_n = c->tie_n;
    a.tie_cap = c->tie_cap;
    a.step_no = c->step_no;
    a.fb1t = (c->use_fb1t && c->use_gen) ? 1 : 0;
    a.k8_long = (!c->k8_warp && !c->k8_block) ? c->k8_long : 0;
    a.fbs = c->fbs;
    for (int k = 0; k < 3; ++k)
    {
        a.fbs_off[k] = c->fbs_off[k];
        a.fbs_cap[k] = c->fbs_cap[k];
    }
    for (int i = 0; i < kL; ++i)
    {
        a.frc_off[i] = 2 * c->frc_off[i];
        a.frc_x0[i] = c->frc_x0[i];
        a.frc_y0[i] = c->frc_y0[i];
        a.frc_nx[i] = c->frc_nx[i];
        a.frc_ny[i] = c->frc_ny[i];
    }
    return a;
}

int grid_for(mrlbm_ctx* c, long long n, int threads = 256)
{
    long long b = (n + threads - 1) / threads;
    if (b < 1)
        b = 1;
    if (b > c->grid_cap)
        b = c->grid_cap;
    return static_cast<int>(b);
}

void kmark(mrlbm_ctx* c, const char* name, int level);


void kmark(mrlbm_ctx* c, const char* name, int level)
{
    if (c->profiling != 1)
        return;
    if (c->kn >= static_cast<int>(c->kev.size()))
    {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->kev.push_back(e);
        c->klabel.emplace_back();
    }
    cudaEventRecord(c->kev[c->kn], c->stream);
    c->klabel[c->kn] = {name, level};
    ++c->kn;
}

// block ranges of a multi-level launch over levels [m0, m1]
template <class Blocks>
LGrid make_lgrid(mrlbm_ctx* c, int m0, int m1, Blocks&& blocks, int* total)
{
    LGrid lg{};
    lg.m0 = m0;
    lg.nl = m1 - m0 + 1;
    lg.start[0] = 0;
    for (int i = 0; i < lg.nl; ++i)
        lg.start[i + 1] = lg.start[i] + static_cast<int>(blocks(m0 + i - c->J0));
    *total = lg.start[lg.nl];
    return lg;
}

TileP tiles_of(mrlbm_ctx* c)
{
    TileP t{};
    for (int i = 0; i < c->nlev; ++i)
        t.t[i] = c->tiles[i];
    return t;
}

// compaction of every level of tree version v: tile counts, per-level scans, scatter
void launch_compaction_all(mrlbm_ctx* c, const Geo& g, Flags fl, Tree tv)
{
    TileP tp = tiles_of(c);
    int nb = 0;
    LGrid lt = make_lgrid(c, c->J0, c->J1, [&](int li) { return c->ntiles[li]; }, &nb);
    k_tile_count_ml<<<nb, kTileThreads, 0, c->stream>>>(g, fl, tp, lt);
    kmark(c, "k_tile_count", -1);
    int ns = 0;
    LGrid ls = make_lgrid(c, c->J0, c->J1, [&](int) { return 1; }, &ns);
    k_tile_scan_ml<<<ns, 1024, 0, c->stream>>>(g, tp, tv, ls);
    kmark(c, "k_tile_scan", -1);
    k_tile_scatter_ml<<<nb, kTileThreads, 0, c->stream>>>(g, fl, tp, tv, lt);
    kmark(c, "k_tile_scatter", -1);
    c->kcount += 3;
}

void phase_mark(mrlbm_ctx* c, int k)
{
    if (c->profiling)
        cudaEventRecord(c->ev[k], c->stream);
}

template <int D, int Q, int BS, int EQ, bool GEN>
void enqueue_step(mrlbm_ctx* c)
{
    const int o = c->cur, n = 1 - c->cur;
    const Geo& g = c->geo;
    Tree to = tree_of(c, o), tn = tree_of(c, n);
    // S = state f* (read, transferred in place), T = stream output (next state)
    Fld Sf = fld_of(c, c->curf), Tf = fld_of(c, 1 - c->curf);
    Flags fl = flags_of(c, n);
    Aux aux = aux_of(c);
    cudaStream_t s = c->stream;
    const int T = 256;
    c->kcount = 0;
    c->kn = 0;
    int nb = 0;
    if (c->frc)
        cudaMemsetAsync(c->frc, 0, sizeof(double) * 2 * c->frc_n, s);
    {
        LGrid lz = make_lgrid(c, c->J0, c->J1, [&](int li) { return grid_for(c, g.cap[li] / 16 + 1, T); }, &nb);
        c->kcount++;
        // the per-step flags are first touched by the details: zeroing runs beside the K1 projections
        const bool fz = c->fork_stream && c->profiling != 1 && !c->fuse_pd;
        if (fz)
        {
            cudaEventRecord(c->ev_fork, s);
            cudaStreamWaitEvent(c->side[0], c->ev_fork, 0);
        }
        k_zero_flags<<<nb, T, 0, fz ? c->side[0] : s>>>(g, fl, lz, c->fbc);
        if (fz)
            cudaEventRecord(c->ev_join[0], c->side[0]);
        kmark(c, "k_zero_flags", -1);
    }
    phase_mark(c, 0);
    if (c->fuse_pd)
    {
        // K1 + K2 fused per level, bottom-up (the details phase is folded into "project")
        for (int m = c->J1 - 1; m >= c->J0; --m)
        {
            c->kcount++;
            k_proj_details<D, Q><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, to, Sf, fl, c->sch, m, aux);
            kmark(c, "k_proj_details", m);
        }
        phase_mark(c, 1);
    }
    else
    {
        // K1 projection of the old tree (bottom-up)
        for (int m = c->J1 - 1; m >= c->J0; --m)
            { c->kcount++; k_project<D, Q><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, to, Sf, m, aux);  kmark(c, "k_project", m); }
        phase_mark(c, 1);
        if (c->fork_stream && c->profiling != 1)
            cudaStreamWaitEvent(s, c->ev_join[0], 0); // k_zero_flags
        // K2 details + flags
        LGrid lg = make_lgrid(c, c->J0, c->J1 - 1, [&](int li) { return grid_for(c, g.cap[li], T); }, &nb);
        c->kcount++;
        k_details<D, Q><<<nb, T, 0, s>>>(g, to, Sf, fl, c->sch, lg, aux);
        kmark(c, "k_details", -1);
    }
    phase_mark(c, 2);
    // K3 closure, enlargement, grading
    auto vec_ok = [&](int m) { return D == 2 && g.ny[m - c->J0] % 16 == 0 && g.lny[m - c->J0] >= 0; };
    for (int m = c->J1 - 1; m > c->J0; --m)
    {
        c->kcount++;
        if (vec_ok(m - 1))
            k_closure_v<<<grid_for(c, g.cap[m - 1 - c->J0] / 16, T), T, 0, s>>>(g, fl, m);
        else
            k_closure<D><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, to, fl, m);
        kmark(c, "k_closure", m);
    }
    {
        // H(a): levels [J0, me) scatter from the kept parents, [me, J1) gather 16 cells per thread
        int me = c->J1;
        for (int m = c->J1 - 1; m >= c->J0 && vec_ok(m); --m)
            me = m;
        if (me > c->J0)
        {
            LGrid lg = make_lgrid(c, c->J0, me - 1, [&](int li) { return grid_for(c, g.cap[li], T); }, &nb);
            c->kcount++;
            k_enlarge<D><<<nb, T, 0, s>>>(g, to, fl, c->sch, lg, c->emask);
            kmark(c, "k_enlarge", -1);
        }
        if (me < c->J1)
        {
            LGrid lg = make_lgrid(c, me, c->J1 - 1, [&](int li) { return grid_for(c, g.cap[li] / 16, T); }, &nb);
            c->kcount++;
            k_enlarge_v<<<nb, T, 0, s>>>(g, fl, lg, c->emask);
            kmark(c, "k_enlarge", -1);
        }
    }
    for (int m = c->J1 - 1; m > c->J0; --m)
    {
        c->kcount++;
        if (vec_ok(m))
            k_grade_v<<<grid_for(c, g.cap[m - c->J0] / 16, T), T, 0, s>>>(g, fl, m);
        else
            k_grade<D><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, fl, m);
        kmark(c, "k_grade", m);
    }
    phase_mark(c, 3);
    // K4 kinds, fallback flags, reconstruction bands, ghosts, compaction
    // levels [J0, mv) use the scalar dense kernels, [mv, J1] the 16-cell vector ones
    int mv = c->J1 + 1;
    for (int m = c->J1; m >= c->J0 && vec_ok(m); --m)
        mv = m;
    auto blocks_s = [&](int li) { return grid_for(c, g.cap[li], T); };
    auto blocks_v = [&](int li) { return grid_for(c, g.cap[li] / 16, T); };
    if (mv > c->J0)
    {
        LGrid lg = make_lgrid(c, c->J0, mv - 1, blocks_s, &nb);
        c->kcount++;
        k_kinds<D><<<nb, T, 0, s>>>(g, fl, lg);
        kmark(c, "k_kinds", -1);
    }
    if (mv <= c->J1)
    {
        LGrid lg = make_lgrid(c, mv, c->J1, blocks_v, &nb);
        c->kcount++;
        k_kinds_v<<<nb, T, 0, s>>>(g, fl, lg);
        kmark(c, "k_kinds_v", -1);
    }
    // Pass 1 of the ghost dilation reads R membership only (fixed by the kinds kernels; the fallback
    // bit and the band marks never touch the leaf / internal bits) and writes its own scratch (keep,
    // free after K3): it runs beside the fallback classification, the lists and the band marking.
    // Pass 2 marks 0 -> K_VIRT with byte stores, like the band marking: both only ever write
    // K_VIRT into bytes without a leaf / internal bit, so they commute.  The whole ghost
    // dilation runs beside classification, lists and bands; the compaction waits for both.
    const bool fgr = c->fork_stream && c->profiling != 1;
    cudaStream_t sGr = fgr ? c->side[2] : s;
    auto ghost_rows = [&]() {
        if (mv > c->J0 && D == 2)
        {
            LGrid lg = make_lgrid(c, c->J0, mv - 1, blocks_s, &nb);
            c->kcount++;
            k_ghost_rows<D><<<nb, T, 0, sGr>>>(g, fl, lg);
            kmark(c, "k_ghost_rows", -1);
        }
        if (mv <= c->J1)
        {
            LGrid lg = make_lgrid(c, mv, c->J1, blocks_v, &nb);
            c->kcount++;
            k_ghost_rows_v<<<nb, T, 0, sGr>>>(g, fl, lg);
            kmark(c, "k_ghost_rows_v", -1);
        }
    };
    auto ghost_marks = [&]() {
        if (mv > c->J0)
        {
            LGrid lg = make_lgrid(c, c->J0, mv - 1, blocks_s, &nb);
            c->kcount++;
            k_ghost<D><<<nb, T, 0, sGr>>>(g, fl, lg);
            kmark(c, "k_ghost", -1);
        }
        if (mv <= c->J1)
        {
            LGrid lg = make_lgrid(c, mv, c->J1, blocks_v, &nb);
            c->kcount++;
            k_ghost_v<<<nb, T, 0, sGr>>>(g, fl, lg);
            kmark(c, "k_ghost_v", -1);
        }
    };
    if (fgr)
    {
        cudaEventRecord(c->ev_fork, s);
        cudaStreamWaitEvent(sGr, c->ev_fork, 0);
        ghost_rows();
        ghost_marks();
        cudaEventRecord(c->ev_join[2], sGr);
    }
    if (mv > c->J0)
    {
        LGrid lg = make_lgrid(c, c->J0, mv - 1, blocks_s, &nb);
        c->kcount++;
        k_fallback<D><<<nb, T, 0, s>>>(g, fl, lg, aux);
        kmark(c, "k_fallback", -1);
    }
    if (mv <= c->J1)
    {
        LGrid lg = make_lgrid(c, mv, c->J1, blocks_v, &nb);
        c->kcount++;
        k_fallback_v<<<nb, T, 0, s>>>(g, fl, lg, aux);
        kmark(c, "k_fallback_v", -1);
    }
    if (c->J1 - 2 >= c->J0)
    {
        LGrid ld = make_lgrid(c, c->J0, c->J1 - 2, [&](int li) {
            const long long nt = D == 1 ? (g.nx[li] + 255) / 256 : (long long)((g.nx[li] + 15) / 16) * ((g.ny[li] + 15) / 16);
            return static_cast<int>(std::min<long long>(std::max<long long>(nt, 1), 148 * 4));
        }, &nb);
        c->kcount++;
        k_list_deep<D><<<nb, 256, 0, s>>>(g, fl, ld, aux);
        kmark(c, "k_list_deep", -1);
    }
    // the gap-1 list reads leaf kinds and fallback masks only (band and ghost marking never change a
    // leaf byte's value): it runs beside k_list_deep / k_band / the ghost passes
    const bool fl1 = c->fork_stream && c->profiling != 1;
    bool fl1_used = false;
    if (GEN && c->use_fb1t && c->J1 > c->J0)
    {
        c->kcount++;
        if (fl1)
        {
            cudaEventRecord(c->ev_fork, s);
            cudaStreamWaitEvent(c->side[1], c->ev_fork, 0);
            fl1_used = true;
        }
        k_list_fb1<D><<<c->grid_cap, 256, 0, fl1 ? c->side[1] : s>>>(g, fl, aux);
        if (fl1)
            cudaEventRecord(c->ev_join[1], c->side[1]);
        kmark(c, "k_list_fb1", -1);
    }
    { c->kcount++; k_band<D><<<c->grid_cap, 256, 0, s>>>(g, fl, aux);  kmark(c, "k_band", -1); }
    if (fgr)
        cudaStreamWaitEvent(s, c->ev_join[2], 0);
    else
    {
        ghost_rows();
        ghost_marks();
    }
    launch_compaction_all(c, g, fl, tn);
    if (fl1_used)
        cudaStreamWaitEvent(s, c->ev_join[1], 0); // k_list_fb1
    phase_mark(c, 4);
    // K5 transfer (top-down), K6 projection of the new tree, virtual values (top-down)
    for (int m = c->J0; m <= c->J1; ++m)
        { c->kcount++; k_transfer<D, Q><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, to, tn, Sf, m, aux);  kmark(c, "k_transfer", m); }
    for (int m = c->J1 - 1; m >= c->J0; --m)
        { c->kcount++; k_project_new<D, Q><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, to, tn, Sf, m, c->dirty_d);  kmark(c, "k_project_new", m); }
    for (int m = c->J0 + 1; m <= c->J1; ++m)
        { c->kcount++; k_virtual<D, Q><<<grid_for(c, g.cap[m - c->J0], T), T, 0, s>>>(g, tn, Sf, m, aux);  kmark(c, "k_virtual", m); }
    phase_mark(c, 5);
    // K7/K8 stream + collide (+ obstacle) on every new leaf.  Fork: every launch below reads the
    // transferred state (Sf) and writes its own leaves of Tf; only MODE 1 (collision of the deep-gap
    // fallback leaves) reads what K8 wrote.  Not in profiling mode (the per-kernel events assume one stream).
    const bool forked = c->fork_stream && c->profiling != 1;
    cudaStream_t sK8L = s, sRim = s, sFb1t = s, sL12 = s, sCoarse = s;
    if (forked)
    {
        cudaEventRecord(c->ev_fork, s);
        for (int i = 0; i < 5; ++i)
            cudaStreamWaitEvent(c->side[i], c->ev_fork, 0);
        sK8L = c->side[0];
        sRim = c->side[1];
        sFb1t = c->side[2];
        sL12 = c->side[3];
        sCoarse = c->side[4];
    }
    c->kcount++;
    if (c->k8_warp)
        k_stream_fallback<D><<<c->grid_cap, 256, 0, s>>>(g, tn, Tf, Sf, fl, c->sch, aux);
    else if (c->k8_block)
        k_stream_fallback_b<D><<<c->grid_cap, 32 * Q, 0, s>>>(g, tn, Tf, Sf, c->sch, aux);
    else if (c->k8_occ == 3)
        k_stream_fallback_t<D, 3><<<c->grid_cap, 256, 0, s>>>(g, tn, Tf, Sf, c->sch, aux);
    else if (c->k8_occ == 4)
        k_stream_fallback_t<D, 4><<<c->grid_cap, 256, 0, s>>>(g, tn, Tf, Sf, c->sch, aux);
    else if (c->k8_occ == 5)
        k_stream_fallback_t<D, 5><<<c->grid_cap, 256, 0, s>>>(g, tn, Tf, Sf, c->sch, aux);
    else if (c->k8_occ == 6)
        k_stream_fallback_t<D, 6><<<c->grid_cap, 256, 0, s>>>(g, tn, Tf, Sf, c->sch, aux);
    else
        k_stream_fallback_t<D, 2><<<c->grid_cap, 256, 0, s>>>(g, tn, Tf, Sf, c->sch, aux);
    kmark(c, "k_stream_fallback", -1);
    if (aux.k8_long > 0 && c->J1 - aux.k8_long >= c->J0)
    {
        c->kcount++;
        k_stream_fallback_long<D><<<c->grid_cap, 256, 0, sK8L>>>(g, tn, Tf, Sf, c->sch, aux);
        kmark(c, "k_stream_fallback_long", -1);
    }
    CollC<Q, BS> cc;
    for (int i = 0; i < Q; ++i)
        for (int j = 0; j < BS; ++j)
        {
            const int col = (i / BS) * BS + j;
            cc.M[i * BS + j] = c->sc.M[i * Q + col];
            cc.Mi[i * BS + j] = c->sc.Minv[i * Q + col];
        }
    // force tracking (config 5 diagnostics) runs separately compiled variants, so the
    // default kernels carry no extra code
    constexpr bool kObs = EQ == MRLBM_EQ_NS_D2Q9 && D == 2;
    const bool frc = kObs && c->frc != nullptr;
    // thread-per-leaf fallback path (generated code): gap-1 fallback leaves in K7 MODE 2
    // (slot scan) and MODE 3 (listed boundary-rim ones), gap-0 fallback leaves in MODE 5
    // (listed); otherwise k_fb1 scans the gap-1 leaves and MODE 1 all levels
    const bool tpl = GEN && c->use_fb1t;
    if (c->J1 > c->J0)
    {
        if (!tpl)
        {
            c->kcount++;
            if (frc)
                k_fb1<D, Q, BS, EQ, GEN, kObs><<<c->grid_cap, 32 * Q, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, aux, cc);
            else
                k_fb1<D, Q, BS, EQ, GEN><<<c->grid_cap, 32 * Q, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, aux, cc);
            kmark(c, "k_fb1", -1);
        }
        else if (!c->rim_tpl)
        {
            // the listed boundary-rim gap-1 leaves: Q warps per batch, compact generic loops
            c->kcount++;
            if (frc)
                k_fb1<D, Q, BS, EQ, false, kObs><<<c->grid_cap, 32 * Q, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, aux, cc);
            else
                k_fb1<D, Q, BS, EQ, false><<<c->grid_cap, 32 * Q, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, aux, cc);
            kmark(c, "k_fb1_rim", -1);
        }
        if constexpr (GEN)
        if (tpl)
        {
            LGrid l2 = make_lgrid(c, c->J1 - 1, c->J1 - 1, [&](int li) { return grid_for(c, g.cap[li], 256); }, &nb);
            c->kcount += 2;
            if (frc)
                k_stream_collide<D, Q, BS, EQ, GEN, 2, 1, kObs><<<nb, 256, 0, sFb1t>>>(g, tn, Tf, Sf, fl, c->sch, l2, aux, cc);
            else
                k_stream_collide<D, Q, BS, EQ, GEN, 2, 1><<<nb, 256, 0, sFb1t>>>(g, tn, Tf, Sf, fl, c->sch, l2, aux, cc);
            kmark(c, "k_fb1t", -1);
            if (c->rim_tpl)
            {
                LGrid l3 = make_lgrid(c, c->J1 - 1, c->J1 - 1, [&](int) { return 148; }, &nb);
                if (frc)
                    k_stream_collide<D, Q, BS, EQ, GEN, 3, 1, kObs><<<nb, 256, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, l3, aux, cc);
                else
                    k_stream_collide<D, Q, BS, EQ, GEN, 3, 1><<<nb, 256, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, l3, aux, cc);
                kmark(c, "k_fb1_rim", -1);
            }
            else
                c->kcount--;
        }
    }
    {
        LGrid lg = make_lgrid(c, c->J0, c->J1, [&](int li) { return grid_for(c, g.cap[li], 256); }, &nb);
        c->kcount++;
        if constexpr (GEN)
        {
            // the generated path in two register budgets: the finest level (gap 0) alone,
            // then every coarser level (gap classes 1 and >= 2)
            LGrid l0 = make_lgrid(c, c->J1, c->J1, [&](int li) { return grid_for(c, g.cap[li], 256); }, &nb);
            if (frc)
                k_stream_collide<D, Q, BS, EQ, GEN, 0, 0, kObs><<<nb, 256, 0, sL12>>>(g, tn, Tf, Sf, fl, c->sch, l0, aux, cc);
            else
                k_stream_collide<D, Q, BS, EQ, GEN, 0, 0><<<nb, 256, 0, sL12>>>(g, tn, Tf, Sf, fl, c->sch, l0, aux, cc);
            kmark(c, "k_stream_collide", c->J1);
            if (c->J1 > c->J0)
            {
                LGrid l1 = make_lgrid(c, c->J0, c->J1 - 1, [&](int li) { return grid_for(c, g.cap[li], 256); }, &nb);
                c->kcount++;
                if (frc)
                    k_stream_collide<D, Q, BS, EQ, GEN, 0, 1, kObs><<<nb, 256, 0, sCoarse>>>(g, tn, Tf, Sf, fl, c->sch, l1, aux, cc);
                else
                    k_stream_collide<D, Q, BS, EQ, GEN, 0, 1><<<nb, 256, 0, sCoarse>>>(g, tn, Tf, Sf, fl, c->sch, l1, aux, cc);
                kmark(c, "k_stream_collide", -1);
            }
        }
        else
        {
            if (frc)
                k_stream_collide<D, Q, BS, EQ, GEN, 0, -1, kObs><<<nb, 256, 0, sL12>>>(g, tn, Tf, Sf, fl, c->sch, lg, aux, cc);
            else
                k_stream_collide<D, Q, BS, EQ, GEN, 0, -1><<<nb, 256, 0, sL12>>>(g, tn, Tf, Sf, fl, c->sch, lg, aux, cc);
            kmark(c, "k_stream_collide", -1);
        }
        // MODE 1: deep-gap fallback leaves (collide K8's output) by slot scan, and with
        // !tpl also the gap-0 ones; with tpl the gap-0 ones come from their list (MODE 5)
        const int mtop = tpl ? c->J1 - 2 : c->J1;
        if (mtop >= c->J0)
        {
            LGrid lf = make_lgrid(c, c->J0, mtop, [&](int li) { return grid_for(c, g.cap[li] / 8, 256); }, &nb);
            c->kcount++;
            if (forked)
            {
                // K8's long-rim launch ran on its own stream: its leaves are collided here
                cudaEventRecord(c->ev_join[0], sK8L);
                cudaStreamWaitEvent(s, c->ev_join[0], 0);
            }
            if (frc)
                k_stream_collide<D, Q, BS, EQ, GEN, 1, -1, kObs><<<nb, 256, 0, s>>>(g, tn, Tf, Sf, fl, c->sch, lf, aux, cc);
            else
                k_stream_collide<D, Q, BS, EQ, GEN, 1, -1><<<nb, 256, 0, s>>>(g, tn, Tf, Sf, fl, c->sch, lf, aux, cc);
            kmark(c, "k_stream_collide_fb", -1);
        }
        if constexpr (GEN)
        if (tpl)
        {
            LGrid l5 = make_lgrid(c, c->J1, c->J1, [&](int) { return 148; }, &nb);
            c->kcount++;
            if (frc)
                k_stream_collide<D, Q, BS, EQ, GEN, 5, -1, kObs><<<nb, 256, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, l5, aux, cc);
            else
                k_stream_collide<D, Q, BS, EQ, GEN, 5, -1><<<nb, 256, 0, sRim>>>(g, tn, Tf, Sf, fl, c->sch, l5, aux, cc);
            kmark(c, "k_stream_collide_fb0", -1);
        }
    }
    if (forked)
        for (int i = 0; i < 5; ++i)
        {
            cudaEventRecord(c->ev_join[i], c->side[i]);
            cudaStreamWaitEvent(s, c->ev_join[i], 0);
        }
    { c->kcount++; k_count_updates<<<1, 32, 0, s>>>(c->cnt[n], c->nlev, c->upd, c->step_no);  kmark(c, "k_count_updates", -1); }
    if (c->frc)
        { c->kcount++; k_force_sum<<<1, 1024, 0, s>>>(c->frc, c->frc_n, c->fhist, c->fhn, c->fcap);  kmark(c, "k_force_sum", -1); }
    phase_mark(c, 6);
    c->kernels_per_step = c->kcount;
}

using StepFn = void (*)(mrlbm_ctx*);

// The generated code's compile-time constants hold for this scheme: the gap-0 / gap-1
// table weights (table order) and the zero / +-1 pattern of M and M^-1.
bool gen_constants_match(const mrlbm_scheme_spec* sc, int nlev, const std::vector<int2>& idx,
                         const std::vector<double>& w)
{
    const double* gw[2] = {nullptr, nullptr};
    int gn[2] = {0, 0};
    const char* pat[2] = {nullptr, nullptr};
#define GEN_CASE(N)                                                                                                    \
    case N:                                                                                                            \
        gw[0] = gen_w_EQ##N##_g0;                                                                                      \
        gn[0] = static_cast<int>(sizeof(gen_w_EQ##N##_g0) / sizeof(double));                                           \
        gw[1] = gen_w_EQ##N##_g1;                                                                                      \
        gn[1] = static_cast<int>(sizeof(gen_w_EQ##N##_g1) / sizeof(double));                                           \
        pat[0] = gen_pat_EQ##N##_M;                                                                                    \
        pat[1] = gen_pat_EQ##N##_Minv;                                                                                 \
        break;
    switch (sc->equilibrium)
    {
        GEN_CASE(1)
        GEN_CASE(2)
        GEN_CASE(3)
        GEN_CASE(4)
        GEN_CASE(5)
    default:
        return false;
    }
#undef GEN_CASE
    const int q = sc->q, bs = q / sc->nblocks;
    for (int gp = 0; gp < 2 && gp < nlev; ++gp)
    {
        const int b = idx[gp * 2 * q].x;
        const int2 last = idx[gp * 2 * q + 2 * q - 1];
        if (last.x + last.y - b != gn[gp])
            return false;
        for (int e = 0; e < gn[gp]; ++e)
            if (w[b + e] != gw[gp][e])
                return false;
    }
    for (int k = 0; k < 2; ++k)
    {
        const double* A = k == 0 ? sc->M : sc->Minv;
        if (static_cast<int>(std::strlen(pat[k])) != q * bs)
            return false;
        for (int i = 0; i < q; ++i)
            for (int c = 0; c < bs; ++c)
            {
                const double v = A[i * q + (i / bs) * bs + c];
                const char ch = pat[k][i * bs + c];
                if ((ch == '0' && v != 0.0) || (ch == '+' && v != 1.0) || (ch == '-' && v != -1.0))
                    return false;
            }
        // block-diagonal: nothing outside the blocks
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < q; ++j)
                if (j / bs != i / bs && A[i * q + j] != 0.0)
                    return false;
    }
    return true;
}

// the generated stream path applies when the velocities are exactly the built-in
// set of the equilibrium kind (the order csrc/host_configs.cpp uses)
bool builtin_velocities(const mrlbm_scheme_spec* sc)
{
    static const int d2q4[4][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    static const int d2q9[9][2] = {{0, 0}, {1, 0}, {0, 1}, {-1, 0}, {0, -1}, {1, 1}, {-1, 1}, {-1, -1}, {1, -1}};
    for (int h = 0; h < sc->q; ++h)
    {
        int ex = 0, ey = 0;
        switch (sc->equilibrium)
        {
            case MRLBM_EQ_BURGERS_D1Q2: ex = h == 0 ? 1 : -1; break;
            case MRLBM_EQ_EULER_D1Q3X3: ex = (h % 3 == 0) ? 0 : (h % 3 == 1 ? 1 : -1); break;
            case MRLBM_EQ_ADVECTION_D2Q4:
            case MRLBM_EQ_EULER_D2Q4X4: ex = d2q4[h % 4][0]; ey = d2q4[h % 4][1]; break;
            case MRLBM_EQ_NS_D2Q9: ex = d2q9[h][0]; ey = d2q9[h][1]; break;
            default: return false;
        }
        if (sc->eta[h][0] != ex || (sc->d == 2 && sc->eta[h][1] != ey))
            return false;
    }
    return true;
}

StepFn step_fn(int d, int q, int nblocks, int eq, bool gen)
{
#define SF(D, Q, BS, E)                                                                                                    return gen ? enqueue_step<D, Q, BS, E, true> : enqueue_step<D, Q, BS, E, false>;
    if (d == 1 && q == 2 && nblocks == 1 && eq == MRLBM_EQ_BURGERS_D1Q2)
        SF(1, 2, 2, MRLBM_EQ_BURGERS_D1Q2)
    if (d == 1 && q == 9 && nblocks == 3 && eq == MRLBM_EQ_EULER_D1Q3X3)
        SF(1, 9, 3, MRLBM_EQ_EULER_D1Q3X3)
    if (d == 2 && q == 4 && nblocks == 1 && eq == MRLBM_EQ_ADVECTION_D2Q4)
        SF(2, 4, 4, MRLBM_EQ_ADVECTION_D2Q4)
    if (d == 2 && q == 16 && nblocks == 4 && eq == MRLBM_EQ_EULER_D2Q4X4)
        SF(2, 16, 4, MRLBM_EQ_EULER_D2Q4X4)
    if (d == 2 && q == 9 && nblocks == 1 && eq == MRLBM_EQ_NS_D2Q9)
        SF(2, 9, 9, MRLBM_EQ_NS_D2Q9)
#undef SF
    return nullptr;
}

int check_device_errors(mrlbm_ctx* ctx)
{
    int e[4] = {0, 0, 0, 0};
    CU(cudaMemcpyAsync(e, ctx->err, sizeof(e), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (e[0] || e[2])
        return set_err(ctx, MRLBM_ERR_CAPACITY,
                       "mesh invariant violated: unresolved stencils=" + std::to_string(e[0]) +
                           " inconsistencies=" + std::to_string(e[2]));
    if (e[1])
        return set_err(ctx, MRLBM_ERR_NUMERIC, "non-finite populations after collision: " + std::to_string(e[1]));
    return MRLBM_OK;
}

} // namespace

extern "C" {

static int init_obstacle(mrlbm_ctx* ctx);

int mrlbm_create(const mrlbm_scheme_spec* sc, const mrlbm_run_config* rc, mrlbm_ctx** out)
{
    *out = nullptr;
    mrlbm_ctx* ctx = nullptr;
    if (!sc || !rc)
        return MRLBM_ERR_CONFIG;
    if (sc->d == 3)
    {
        ctx = new mrlbm_ctx();
        const int st3 = mrlbm_b200::e3_create(sc, rc, &ctx->e3, ctx->err_msg);
        if (st3 != MRLBM_OK)
        {
            delete ctx;
            return st3;
        }
        ctx->sc = *sc;
        ctx->rc = *rc;
        ctx->D = 3;
        ctx->q = sc->q;
        ctx->J0 = rc->j_min;
        ctx->J1 = rc->j_max;
        ctx->nlev = ctx->J1 - ctx->J0 + 1;
        *out = ctx;
        return MRLBM_OK;
    }
    if (sc->d < 1 || sc->d > 2 || !step_fn(sc->d, sc->q, sc->nblocks, sc->equilibrium, false))
        return MRLBM_ERR_CONFIG;
    if (rc->j_min < 0 || rc->j_max <= rc->j_min || rc->j_max - rc->j_min + 1 > kL)
        return MRLBM_ERR_CONFIG;
    if (rc->gamma != 1 || rc->graduation != 1 || sc->nblocks < 1 || sc->q % sc->nblocks)
        return MRLBM_ERR_CONFIG;
    for (int i = 0; i < sc->d; ++i)
        if ((rc->bc_kind[2 * i] == MRLBM_BC_PERIODIC) != (rc->bc_kind[2 * i + 1] == MRLBM_BC_PERIODIC))
            return MRLBM_ERR_CONFIG;
    ctx = new mrlbm_ctx();
    ctx->sc = *sc;
    ctx->rc = *rc;
    ctx->D = sc->d;
    ctx->q = sc->q;
    ctx->J0 = rc->j_min;
    ctx->J1 = rc->j_max;
    ctx->nlev = ctx->J1 - ctx->J0 + 1;
    Geo& g = ctx->geo;
    g.d = ctx->D;
    g.q = ctx->q;
    g.J0 = ctx->J0;
    g.J1 = ctx->J1;
    g.nlev = ctx->nlev;
    g.per0 = rc->bc_kind[0] == MRLBM_BC_PERIODIC;
    g.per1 = ctx->D == 2 && rc->bc_kind[2] == MRLBM_BC_PERIODIC;
    // 2D values are stored in 2x2 sibling blocks (vix): even level extents
    if (ctx->D == 2 && ((rc->base_cells[0] & 1) || (rc->base_cells[1] & 1)))
    {
        delete ctx;
        return MRLBM_ERR_CONFIG;
    }
    for (int li = 0; li < ctx->nlev; ++li)
    {
        const long long nx = rc->base_cells[0] << li;
        const long long ny = ctx->D == 2 ? (rc->base_cells[1] << li) : 1;
        if (nx * ny >= (1LL << 31))
        {
            delete ctx;
            return MRLBM_ERR_CONFIG;
        }
        g.nx[li] = static_cast<int>(nx);
        g.ny[li] = static_cast<int>(ny);
        g.lny[li] = (ny & (ny - 1)) == 0 ? __builtin_ctzll(static_cast<unsigned long long>(ny)) : -1;
        g.cap[li] = nx * ny;
    }
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce != cudaSuccess)
    {
        *out = nullptr;
        delete ctx;
        return MRLBM_ERR_CUDA;
    }
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, dev);
    ctx->grid_cap = prop.multiProcessorCount * 8;
    int st = [&]() -> int
    {
        CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        for (int i = 0; i < 5; ++i)
        {
            CU(cudaStreamCreateWithFlags(&ctx->side[i], cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&ctx->ev_join[i], cudaEventDisableTiming));
        }
        for (int v = 0; v < 2; ++v)
        {
            CU(cudaMalloc(&ctx->cnt[v], sizeof(int) * 4 * kL));
            CU(cudaMemset(ctx->cnt[v], 0, sizeof(int) * 4 * kL));
        }
        long long total_cells = 0;
        for (int li = 0; li < ctx->nlev; ++li)
        {
            const long long n = g.cap[li];
            total_cells += n;
            for (int v = 0; v < 2; ++v)
            {
                CU(cudaMalloc(&ctx->cells[v][li], sizeof(int32_t) * n));
                CU(cudaMalloc(&ctx->skind[v][li], n));
                CU(cudaMalloc(&ctx->kind2[v][li], n));
                CU(cudaMemset(ctx->kind2[v][li], 0, n));
                CU(cudaMalloc(&ctx->F[v][li], sizeof(double) * n * ctx->q));
                CU(cudaMemset(ctx->F[v][li], 0, sizeof(double) * n * ctx->q));
            }
            CU(cudaMalloc(&ctx->rn[li], n));
            CU(cudaMalloc(&ctx->keep[li], n));
            CU(cudaMalloc(&ctx->fbmd[li], sizeof(unsigned) * n));
            CU(cudaMalloc(&ctx->fbdd[li], sizeof(unsigned) * n));
            ctx->ntiles[li] = (n + kTile - 1) / kTile;
            CU(cudaMalloc(&ctx->tiles[li], sizeof(int) * 3 * ctx->ntiles[li]));
            // load / read-back staging (coordinates and linear indices of one level),
            // allocated with the context so the first load or read pays no allocation
            CU(cudaMalloc(&ctx->ld_idx[li], sizeof(int32_t) * ctx->D * n));
            CU(cudaMalloc(&ctx->ld_lin[li], sizeof(int32_t) * n));
        }
        CU(cudaMalloc(&ctx->ld_bad, sizeof(int)));
        CU(cudaMalloc(&ctx->rdcnt, sizeof(int) * 4));
        ctx->fbcap = total_cells;
        CU(cudaMalloc(&ctx->dirty_d, sizeof(uint8_t*) * kL));
        CU(cudaMemcpy(ctx->dirty_d, ctx->keep, sizeof(uint8_t*) * kL, cudaMemcpyHostToDevice));
        CU(cudaMalloc(&ctx->fbl, sizeof(int2) * ctx->fbcap));
        CU(cudaMalloc(&ctx->fbm, sizeof(unsigned) * ctx->fbcap));
        CU(cudaMalloc(&ctx->fbdm, sizeof(unsigned) * ctx->fbcap));
        CU(cudaMalloc(&ctx->fbc, sizeof(int) * 8));
        CU(cudaMemset(ctx->fbc, 0, sizeof(int) * 8));
        // segment lists: capacity = the level's cell count (J1 for gap 0, J1-1 for gap 1)
        ctx->fbs_cap[0] = ctx->geo.cap[ctx->nlev - 1];
        ctx->fbs_cap[1] = ctx->nlev > 1 ? ctx->geo.cap[ctx->nlev - 2] : 0;
        ctx->fbs_cap[2] = ctx->fbs_cap[1];
        ctx->fbs_off[0] = 0;
        ctx->fbs_off[1] = ctx->fbs_cap[0];
        ctx->fbs_off[2] = ctx->fbs_cap[0] + ctx->fbs_cap[1];
        CU(cudaMalloc(&ctx->fbs, sizeof(int) * (ctx->fbs_cap[0] + ctx->fbs_cap[1] + ctx->fbs_cap[2] + 1)));
        CU(cudaMalloc(&ctx->err, sizeof(int) * 4));
        CU(cudaMemset(ctx->err, 0, sizeof(int) * 4));
        CU(cudaMalloc(&ctx->upd, sizeof(long long)));
        CU(cudaMemset(ctx->upd, 0, sizeof(long long)));
        CU(cudaMalloc(&ctx->ties, sizeof(mrlbm_tie_record) * ctx->tie_cap));
        CU(cudaMalloc(&ctx->tie_n, sizeof(int)));
        CU(cudaMemset(ctx->tie_n, 0, sizeof(int)));
        CU(cudaMalloc(&ctx->step_no, sizeof(int)));
        CU(cudaMemset(ctx->step_no, 0, sizeof(int)));
        // scheme constants
        SchemeDev h{};
        h.q = sc->q;
        h.nblocks = sc->nblocks;
        h.bs = sc->q / sc->nblocks;
        h.eq = sc->equilibrium;
        h.mu = rc->mu;
        h.lambda = sc->lambda;
        h.eps = rc->epsilon;
        h.obstacle = rc->obstacle;
        h.obs_ns = rc->obstacle_subsamples;
        for (int i = 0; i < sc->q; ++i)
        {
            h.eta[i][0] = sc->eta[i][0];
            h.eta[i][1] = sc->eta[i][1];
            h.s[i] = sc->s[i];
            h.obs_feq[i] = rc->obstacle_feq[i];
            h.opp[i] = -1;
            const int bs = h.bs;
            for (int k = 0; k < sc->q; ++k)
                if (k / bs == i / bs && sc->eta[k][0] == -sc->eta[i][0] && (sc->d == 1 || sc->eta[k][1] == -sc->eta[i][1]))
                {
                    h.opp[i] = k;
                    break;
                }
            for (int j = 0; j < sc->q; ++j)
            {
                h.M[i * sc->q + j] = sc->M[i * sc->q + j];
                h.Minv[i * sc->q + j] = sc->Minv[i * sc->q + j];
            }
        }
        for (int k = 0; k < 8; ++k)
            h.eqp[k] = sc->eq_params[k];
        for (int f = 0; f < 4; ++f)
        {
            h.bc_kind[f] = rc->bc_kind[f];
            for (int i = 0; i < sc->q; ++i)
                h.bc_add[f][i] = rc->bc_add[f][i];
        }
        h.origin[0] = rc->origin[0];
        h.origin[1] = rc->origin[1];
        h.obs_c[0] = rc->obstacle_center[0];
        h.obs_c[1] = rc->obstacle_center[1];
        h.obs_r = rc->obstacle_radius;
        CU(cudaMalloc(&ctx->sch, sizeof(SchemeDev)));
        CU(cudaMemcpy(ctx->sch, &h, sizeof(SchemeDev), cudaMemcpyHostToDevice));
        // flattened tables + exactness sets for every gap / population / side
        std::vector<int2> idx, off, pidx, par, upidx, upar, guidx, guoff;
        std::vector<int4> dep, udep;
        std::vector<double> w;
        std::vector<uint8_t> tu;
        std::vector<unsigned short> pmask, umask;
        for (int gp = 0; gp < ctx->nlev; ++gp)
        {
            unsigned short um = 0;
            int4 ub = make_int4(0, 0, 0, 0);
            std::vector<std::pair<int, int>> un;
            std::vector<std::pair<int, int>> gu; // distinct table offsets of this gap
            guidx.push_back(make_int2(static_cast<int>(guoff.size()), 0));
            for (int hh = 0; hh < sc->q; ++hh)
            {
                if (std::abs(sc->eta[hh][0]) > 1 || (sc->d == 2 && std::abs(sc->eta[hh][1]) > 1))
                    return set_err(ctx, MRLBM_ERR_CONFIG, "velocities with |eta_i| > 1 are not supported");
                for (int side = 0; side < 2; ++side)
                {
                    std::vector<TableEntry> t;
                    TableSets ts{};
                    const int rcode = build_stream_table(sc->d, gp, sc->eta[hh], side, t, &ts);
                    if (rcode != MRLBM_OK)
                        return set_err(ctx, rcode, "flattened table construction failed");
                    idx.push_back(make_int2(static_cast<int>(off.size()), static_cast<int>(t.size())));
                    for (const auto& e : t)
                    {
                        off.push_back(make_int2(e.off[0], e.off[1]));
                        w.push_back(e.w);
                        const std::pair<int, int> o(e.off[0], e.off[1]);
                        auto it = std::find(gu.begin(), gu.end(), o);
                        tu.push_back(static_cast<uint8_t>(it - gu.begin()));
                        if (it == gu.end())
                            gu.push_back(o);
                    }
                    const int4 db = make_int4(ts.dep_lo[0], ts.dep_hi[0], ts.dep_lo[1], ts.dep_hi[1]);
                    dep.push_back(db);
                    ub = make_int4(std::min(ub.x, db.x), std::max(ub.y, db.y), std::min(ub.z, db.z), std::max(ub.w, db.w));
                    pidx.push_back(make_int2(static_cast<int>(par.size()), static_cast<int>(ts.par.size())));
                    unsigned short pm = 0;
                    for (const auto& p : ts.par)
                    {
                        if (std::abs(p.first) > 1 || std::abs(p.second) > 1)
                            return set_err(ctx, MRLBM_ERR_CONFIG, "table parent outside the 3^d box");
                        pm |= static_cast<unsigned short>(1u << ((p.first + 1) * 3 + (p.second + 1)));
                    }
                    pmask.push_back(pm);
                    um |= pm;
                    for (const auto& p : ts.par)
                    {
                        par.push_back(make_int2(p.first, p.second));
                        if (std::find(un.begin(), un.end(), p) == un.end())
                            un.push_back(p);
                    }
                }
            }
            guidx.back().y = static_cast<int>(gu.size());
            for (const auto& o : gu)
                guoff.push_back(make_int2(o.first, o.second));
            umask.push_back(um);
            udep.push_back(ub);
            upidx.push_back(make_int2(static_cast<int>(upar.size()), static_cast<int>(un.size())));
            for (const auto& p : un)
                upar.push_back(make_int2(p.first, p.second));
        }
        if (off.empty())
        {
            off.push_back(make_int2(0, 0));
            w.push_back(0.0);
        }
        if (par.empty())
            par.push_back(make_int2(0, 0));
        if (upar.empty())
            upar.push_back(make_int2(0, 0));
        if (guoff.empty())
            guoff.push_back(make_int2(0, 0));
        tu.push_back(0);
        auto up = [&](auto*& dst, const auto& v) -> int
        {
            using T = typename std::decay_t<decltype(v)>::value_type;
            CU(cudaMalloc(&dst, sizeof(T) * v.size()));
            CU(cudaMemcpy(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
            return MRLBM_OK;
        };
        std::vector<int2> etav;
        for (int hh = 0; hh < sc->q; ++hh)
            etav.push_back(make_int2(sc->eta[hh][0], sc->d == 2 ? sc->eta[hh][1] : 0));
        if (up(ctx->pmaskd, pmask) || up(ctx->umaskd, umask) || up(ctx->etad, etav) || up(ctx->tidx, idx) || up(ctx->toff, off) || up(ctx->tw, w) || up(ctx->tdep, dep) || up(ctx->tpidx, pidx) ||
            up(ctx->tpar, par) || up(ctx->udep, udep) || up(ctx->guidx, guidx) || up(ctx->guoff, guoff) || up(ctx->tu, tu) || up(ctx->upidx, upidx) || up(ctx->upar, upar))
            return MRLBM_ERR_CUDA;
        for (auto& e : ctx->ev)
            CU(cudaEventCreate(&e));
        ctx->gen_ok = gen_constants_match(sc, ctx->nlev, idx, w);
        if (rc->obstacle == 1 && sc->d == 2 && sc->equilibrium == MRLBM_EQ_NS_D2Q9)
            return init_obstacle(ctx);
        return MRLBM_OK;
    }();
    if (st != MRLBM_OK)
    {
        const std::string msg = ctx->err_msg;
        mrlbm_destroy(ctx);
        fprintf(stderr, "mrlbm_create: %s\n", msg.c_str());
        return st;
    }
    ctx->use_gen = builtin_velocities(sc) && ctx->gen_ok && std::getenv("MRLBM_NO_GEN") == nullptr;
    ctx->use_fb1t = std::getenv("MRLBM_NO_FB1T") == nullptr;
    ctx->rim_tpl = std::getenv("MRLBM_RIM_TPL") != nullptr;
    ctx->fuse_pd = std::getenv("MRLBM_FUSE_PD") != nullptr;
    ctx->k8_warp = std::getenv("MRLBM_K8_WARP") != nullptr;
    ctx->k8_block = std::getenv("MRLBM_K8_BLOCK") != nullptr;
    ctx->fork_stream = std::getenv("MRLBM_SERIAL_STREAM") == nullptr;
    if (const char* oc = std::getenv("MRLBM_K8_OCC"))
        ctx->k8_occ = std::atoi(oc);
    if (const char* lg = std::getenv("MRLBM_K8_LONG_GAP")) // 0: all deep-gap leaves stay in the thread kernel
        ctx->k8_long = std::max(0, std::atoi(lg));
    for (int h = 0; h < sc->q; ++h)
    {
        const int ex = sc->eta[h][0], ey = sc->d == 2 ? sc->eta[h][1] : 0;
        if (ex == 0 && ey == 0)
            continue;
        for (int dl = 0; dl < (1 << sc->d); ++dl)
        {
            const int dx = sc->d == 1 ? dl : dl >> 1, dy = sc->d == 1 ? 0 : dl & 1;
            const int ox = (dx - ex) >> 1, oy = (dy - ey) >> 1; // floor division
            ctx->emask |= 1u << ((ox + 1) * 3 + (oy + 1));
        }
    }
    *out = ctx;
    return MRLBM_OK;
}

int mrlbm_load_leaves(mrlbm_ctx* ctx, int level, int64_t n, const int32_t* idx, const double* f)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_load_leaves(ctx->e3, level, n, idx, f);
    if (level < ctx->J0 || level > ctx->J1 || n < 0)
        return set_err(ctx, MRLBM_ERR_CONFIG, "load: level out of range");
    const int li = level - ctx->J0;
    if (n > ctx->geo.cap[li])
        return set_err(ctx, MRLBM_ERR_CONFIG, "load: more leaves than cells in the level");
    if (!ctx->ld_idx[li])
    {
        CU(cudaMalloc(&ctx->ld_idx[li], sizeof(int32_t) * ctx->D * ctx->geo.cap[li]));
        CU(cudaMalloc(&ctx->ld_lin[li], sizeof(int32_t) * ctx->geo.cap[li]));
    }
    if (!ctx->ld_bad)
        CU(cudaMalloc(&ctx->ld_bad, sizeof(int)));
    ctx->ld_n[li] = n;
    if (n)
    {
        // synchronous copies: the caller may reuse its buffers on return (pinned buffers go at full link speed)
        CU(cudaMemcpyAsync(ctx->ld_idx[li], idx, sizeof(int32_t) * ctx->D * n, cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemcpyAsync(ctx->F[1][li], f, sizeof(double) * ctx->q * n, cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemsetAsync(ctx->ld_bad, 0, sizeof(int), ctx->stream));
        k_idx_to_lin<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(ctx->ld_idx[li], (int)n, ctx->D, ctx->geo.nx[li],
                                                                 ctx->geo.ny[li], ctx->ld_lin[li], ctx->ld_bad);
        int bad = 0;
        CU(cudaMemcpyAsync(&bad, ctx->ld_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (bad)
            return set_err(ctx, MRLBM_ERR_CONFIG, "load: leaf outside the domain");
    }
    ctx->committed = false;
    return MRLBM_OK;
}

int mrlbm_commit(mrlbm_ctx* ctx)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_commit(ctx->e3);
    const Geo& g = ctx->geo;
    const int v = ctx->cur;
    Flags fl = flags_of(ctx, v);
    ctx->curf = 0;
    for (int li = 0; li < ctx->nlev; ++li)
    {
        CU(cudaMemsetAsync(ctx->keep[li], 0, g.cap[li], ctx->stream));
        CU(cudaMemsetAsync(ctx->rn[li], 0, g.cap[li], ctx->stream));
    }
    CU(cudaMemsetAsync(ctx->err, 0, sizeof(int) * 4, ctx->stream));
    CU(cudaMemsetAsync(ctx->step_no, 0, sizeof(int), ctx->stream));
    CU(cudaMemsetAsync(ctx->tie_n, 0, sizeof(int), ctx->stream));
    auto cleanup = [&]() {};
    int st = [&]() -> int
    {
        for (int li = 0; li < ctx->nlev; ++li)
        {
            const long long n = ctx->ld_n[li];
            if (!n)
                continue;
            const int* dl_li = ctx->ld_lin[li];
            if (ctx->D == 1)
                k_load_mark<1><<<grid_for(ctx, n), 256, 0, ctx->stream>>>(g, fl, dl_li, (int)n, ctx->J0 + li);
            else
                k_load_mark<2><<<grid_for(ctx, n), 256, 0, ctx->stream>>>(g, fl, dl_li, (int)n, ctx->J0 + li);
        }
        for (int m = ctx->J1 - 1; m > ctx->J0; --m)
        {
            if (ctx->D == 1)
                k_closure_dense<1><<<grid_for(ctx, g.cap[m - ctx->J0]), 256, 0, ctx->stream>>>(g, fl, m);
            else
                k_closure_dense<2><<<grid_for(ctx, g.cap[m - ctx->J0]), 256, 0, ctx->stream>>>(g, fl, m);
        }
        {
            int nbk = 0;
            LGrid lg = make_lgrid(ctx, ctx->J0, ctx->J1, [&](int li) { return grid_for(ctx, g.cap[li]); }, &nbk);
            if (ctx->D == 1)
                k_kinds<1><<<nbk, 256, 0, ctx->stream>>>(g, fl, lg);
            else
                k_kinds<2><<<nbk, 256, 0, ctx->stream>>>(g, fl, lg);
            launch_compaction_all(ctx, g, fl, tree_of(ctx, v));
        }
        for (int li = 0; li < ctx->nlev; ++li)
        {
            const long long n = ctx->ld_n[li];
            if (!n)
                continue;
            k_load_scatter<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(ctx->ld_lin[li], ctx->F[1][li], (int)n, ctx->q,
                                                                     ctx->kind2[v][li], ctx->F[0][li], g.cap[li], ctx->err,
                                                                     ctx->D, g.ny[li], g.lny[li]);
        }
        CU(cudaGetLastError());
        int counts[4 * kL];
        CU(cudaMemcpyAsync(counts, ctx->cnt[v], sizeof(int) * 4 * kL, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        for (int li = 0; li < ctx->nlev; ++li)
            if (counts[li * 4] != static_cast<int>(ctx->ld_n[li]))
                return set_err(ctx, MRLBM_ERR_CONFIG, "load: leaves do not form a complete-leaf partition (level " +
                                                          std::to_string(ctx->J0 + li) + ")");
        return check_device_errors(ctx);
    }();
    cleanup();
    if (st != MRLBM_OK)
        return st;
    for (auto& n : ctx->ld_n)
        n = 0;
    for (auto& gph : ctx->graph)
        if (gph)
        {
            cudaGraphExecDestroy(gph);
            gph = nullptr;
        }
    ctx->committed = true;
    return MRLBM_OK;
}

int mrlbm_step(mrlbm_ctx* ctx, int nsteps, mrlbm_step_stats* stats)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_step(ctx->e3, nsteps, stats);
    if (!ctx->committed)
        return set_err(ctx, MRLBM_ERR_STATE, "step before commit");
    StepFn fn = step_fn(ctx->D, ctx->q, ctx->sc.nblocks, ctx->sc.equilibrium, ctx->use_gen);
    // old-tree counts before the last step (per-phase byte model); one small read-back
    // per call, only when statistics are requested
    int old_counts[4 * kL] = {0};
    if (stats && nsteps == 1)
        CU(cudaMemcpy(old_counts, ctx->cnt[ctx->cur], sizeof(old_counts), cudaMemcpyDeviceToHost));
    CU(cudaMemsetAsync(ctx->err, 0, sizeof(int) * 4, ctx->stream));
    CU(cudaEventRecord(ctx->ev[14], ctx->stream));
    double phase[MRLBM_PHASE_COUNT] = {0};
    for (int it = 0; it < nsteps; ++it)
    {
        if (ctx->use_graph && !ctx->profiling)
        {
            cudaGraphExec_t& ge = ctx->graph[ctx->cur];
            if (!ge)
            {
                cudaGraph_t gr;
                CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
                fn(ctx);
                CU(cudaStreamEndCapture(ctx->stream, &gr));
                CU(cudaGraphInstantiate(&ge, gr, 0));
                cudaGraphDestroy(gr);
            }
            CU(cudaGraphLaunch(ge, ctx->stream));
        }
        else
        {
            fn(ctx);
            CU(cudaGetLastError());
            if (ctx->profiling)
            {
                CU(cudaEventSynchronize(ctx->ev[6]));
                const int map_phase[6] = {MRLBM_PHASE_PROJECT, MRLBM_PHASE_DETAILS, MRLBM_PHASE_FLAGS,
                                          MRLBM_PHASE_COMPACT, MRLBM_PHASE_TRANSFER, MRLBM_PHASE_STREAM};
                for (int k = 0; k < 6; ++k)
                {
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, ctx->ev[k], ctx->ev[k + 1]);
                    phase[map_phase[k]] += ms;
                }
                for (int k = 0; k < ctx->kn; ++k)
                {
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, k == 0 ? ctx->ev[0] : ctx->kev[k - 1], ctx->kev[k]);
                    auto& a = ctx->kacc[ctx->klabel[k]];
                    a.first += ms;
                    a.second += 1;
                }
            }
        }
        ctx->cur = 1 - ctx->cur;
        ctx->curf = 1 - ctx->curf;
    }
    CU(cudaEventRecord(ctx->ev[15], ctx->stream));
    const int st = check_device_errors(ctx);
    if (stats)
    {
        std::memset(stats, 0, sizeof(*stats));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[14], ctx->ev[15]);
        stats->ms_total = ms;
        for (int k = 0; k < MRLBM_PHASE_COUNT; ++k)
            stats->ms_phase[k] = phase[k];
        int counts[4 * kL];
        int fb[2];
        long long upd = 0;
        CU(cudaMemcpy(counts, ctx->cnt[ctx->cur], sizeof(counts), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(fb, ctx->fbc, sizeof(fb), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(&upd, ctx->upd, sizeof(upd), cudaMemcpyDeviceToHost));
        stats->levels = ctx->nlev;
        long long nS = 0, nI = 0, nG = 0;
        for (int li = 0; li < ctx->nlev; ++li)
        {
            stats->leaves[li] = counts[li * 4];
            stats->internal[li] = counts[li * 4 + 1];
            stats->virtual_cells[li] = counts[li * 4 + 2];
            nS += counts[li * 4];
            nI += counts[li * 4 + 1];
            nG += counts[li * 4 + 2];
        }
        stats->fallback_leaves = fb[0] + fb[1];
        stats->kernel_launches = ctx->kernels_per_step * nsteps;
        stats->leaf_updates = upd;
        // SURVEY 8d compulsory fp64 model per phase.  Old-tree counts: read before the step
        // when the call ran one step, else approximated by the new ones.  N_G = 0: the
        // virtual (ghost + band) cells this design materialises are not compulsory traffic.
        (void)nG;
        long long oS = 0, oI = 0;
        for (int li = 0; li < ctx->nlev; ++li)
        {
            oS += nsteps == 1 ? old_counts[li * 4] : counts[li * 4];
            oI += nsteps == 1 ? old_counts[li * 4 + 1] : counts[li * 4 + 1];
        }
        const long long b8 = 8LL * ctx->q;
        stats->bytes_phase[MRLBM_PHASE_PROJECT] = b8 * (oS + 2 * oI);
        stats->bytes_phase[MRLBM_PHASE_DETAILS] = b8 * (oS + oI);
        stats->bytes_phase[MRLBM_PHASE_TRANSFER] = b8 * (3 * nS + nI);
        stats->bytes_phase[MRLBM_PHASE_STREAM] = b8 * (2 * nS);
        stats->bytes_stream = stats->bytes_phase[MRLBM_PHASE_STREAM];
        stats->bytes_model = 0;
        for (int k = 0; k < MRLBM_PHASE_COUNT; ++k)
            stats->bytes_model += stats->bytes_phase[k];
    }
    return st;
}

int mrlbm_level_count(mrlbm_ctx* ctx, int level, int64_t* n)
{
    if (!ctx || level < ctx->J0 || level > ctx->J1)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_level_count(ctx->e3, level, n);
    int c = 0;
    CU(cudaMemcpyAsync(&c, ctx->cnt[ctx->cur] + (level - ctx->J0) * 4, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *n = c;
    return MRLBM_OK;
}

int mrlbm_read_leaves(mrlbm_ctx* ctx, int level, int32_t* idx, double* f)
{
    if (!ctx || level < ctx->J0 || level > ctx->J1)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_read_leaves(ctx->e3, level, idx, f);
    const int li = level - ctx->J0;
    for (int k = 0; k < ctx->nlev; ++k)
        if (ctx->ld_n[k])
            return set_err(ctx, MRLBM_ERR_STATE, "read_leaves between load_leaves and commit (staged load pending)");
    int64_t n = 0;
    int st = mrlbm_level_count(ctx, level, &n);
    if (st != MRLBM_OK)
        return st;
    if (n == 0)
        return MRLBM_OK;
    if (!ctx->ld_idx[li])
    {
        CU(cudaMalloc(&ctx->ld_idx[li], sizeof(int32_t) * ctx->D * ctx->geo.cap[li]));
        CU(cudaMalloc(&ctx->ld_lin[li], sizeof(int32_t) * ctx->geo.cap[li]));
    }
    // the step's slots are in value-block order (2D): re-sort the level lexicographically
    // (CellIndex order, cell_set.hpp:333-354) with a row-major compaction of its kinds
    const int32_t* lcells = ctx->cells[ctx->cur][li];
    if (ctx->D == 2)
    {
        if (!ctx->rdcnt)
            CU(cudaMalloc(&ctx->rdcnt, sizeof(int) * 4));
        const long long cap = ctx->geo.cap[li];
        const int ntl = static_cast<int>((cap + kTile - 1) / kTile);
        const uint8_t* kind = ctx->kind2[ctx->cur][li];
        k_tile_count<<<ntl, kTileThreads, 0, ctx->stream>>>(kind, cap, ctx->tiles[li]);
        k_tile_scan<<<1, 1024, 0, ctx->stream>>>(ctx->tiles[li], ntl, ctx->rdcnt);
        k_tile_scatter<<<ntl, kTileThreads, 0, ctx->stream>>>(kind, cap, ctx->tiles[li], ctx->rdcnt, nullptr,
                                                              ctx->ld_lin[li]);
        lcells = ctx->ld_lin[li];
    }
    if (idx)
    {
        k_lin_to_idx<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(lcells, (int)n, ctx->D, ctx->geo.ny[li],
                                                                 ctx->ld_idx[li]);
        CU(cudaMemcpyAsync(idx, ctx->ld_idx[li], sizeof(int32_t) * ctx->D * n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (f)
    {
        double* stage = ctx->F[1 - ctx->curf][li]; // the non-state buffer is free between steps
        k_gather_leaves<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(lcells, (int)n, ctx->q,
                                                                   ctx->F[ctx->curf][li], ctx->geo.cap[li], stage, ctx->D,
                                                                   ctx->geo.ny[li], ctx->geo.lny[li]);
        CU(cudaMemcpyAsync(f, stage, sizeof(double) * ctx->q * n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    return MRLBM_OK;
}

int mrlbm_finest_count(const mrlbm_ctx* ctx, int64_t* n)
{
    if (!ctx || !n)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_finest_count(ctx->e3, n);
    *n = ctx->geo.cap[ctx->nlev - 1];
    return MRLBM_OK;
}

} // extern "C"

namespace {

// f^^ of the current state on every cell of every level, into the non-state buffer
// F[1 - curf] (free between steps; the next step writes before it reads there)
int recon_device(mrlbm_ctx* ctx)
{
    if (!ctx->committed)
        return set_err(ctx, MRLBM_ERR_STATE, "reconstruct before commit");
    const Geo& g = ctx->geo;
    Tree t = tree_of(ctx, ctx->cur);
    Fld S = fld_of(ctx, ctx->curf), R = fld_of(ctx, 1 - ctx->curf);
    cudaStream_t s = ctx->stream;
    for (int m = ctx->J1 - 1; m >= ctx->J0; --m)
    {
        const int nb = grid_for(ctx, g.cap[m - ctx->J0]);
        if (ctx->D == 1)
            k_recon_project<1><<<nb, 256, 0, s>>>(g, t, S, m, ctx->q);
        else
            k_recon_project<2><<<nb, 256, 0, s>>>(g, t, S, m, ctx->q);
    }
    for (int m = ctx->J0; m <= ctx->J1; ++m)
    {
        const int nb = grid_for(ctx, g.cap[m - ctx->J0]);
        if (ctx->D == 1)
            k_recon_level<1><<<nb, 256, 0, s>>>(g, t, S, R, m, ctx->q);
        else
            k_recon_level<2><<<nb, 256, 0, s>>>(g, t, S, R, m, ctx->q);
    }
    CU(cudaGetLastError());
    return MRLBM_OK;
}

} // namespace

extern "C" {

int mrlbm_reconstruct_finest(mrlbm_ctx* ctx, double* f)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return set_err(ctx, MRLBM_ERR_CONFIG, "diagnostics are 1D/2D only");
    if (int st = recon_device(ctx); st != MRLBM_OK)
        return st;
    if (f)
    {
        const int li = ctx->nlev - 1;
        CU(cudaMemcpyAsync(f, ctx->F[1 - ctx->curf][li], sizeof(double) * ctx->q * ctx->geo.cap[li],
                           cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    return MRLBM_OK;
}

int mrlbm_additional_error(mrlbm_ctx* ctx, mrlbm_ctx* ref, const double* row, double* E, double* sums)
{
    if (!ctx || !ref || !row || !E)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3 || ref->e3)
        return set_err(ctx, MRLBM_ERR_CONFIG, "diagnostics are 1D/2D only");
    const int li = ctx->nlev - 1, lr = ref->nlev - 1;
    if (ctx->D != ref->D || ctx->q != ref->q || ctx->J1 != ref->J1 || ctx->geo.nx[li] != ref->geo.nx[lr] ||
        ctx->geo.ny[li] != ref->geo.ny[lr])
        return set_err(ctx, MRLBM_ERR_CONFIG, "additional_error: finest grids differ");
    if (int st = recon_device(ref); st != MRLBM_OK)
        return set_err(ctx, st, std::string("reference: ") + ref->err_msg);
    if (cudaError_t e = cudaStreamSynchronize(ref->stream); e != cudaSuccess)
        return set_err(ctx, MRLBM_ERR_CUDA, std::string("reference stream: ") + cudaGetErrorString(e));
    if (int st = recon_device(ctx); st != MRLBM_OK)
        return st;
    const long long n = ctx->geo.cap[li];
    const int nb = grid_for(ctx, n);
    double* dev = nullptr;
    CU(cudaMallocAsync(&dev, sizeof(double) * (ctx->q + 2 * nb), ctx->stream));
    CU(cudaMemcpyAsync(dev, row, sizeof(double) * ctx->q, cudaMemcpyHostToDevice, ctx->stream));
    k_moment_err<<<nb, 256, 0, ctx->stream>>>(ctx->F[1 - ctx->curf][li], ref->F[1 - ref->curf][lr], n, ctx->q, dev,
                                               n, dev + ctx->q);
    std::vector<double> part(2 * nb);
    CU(cudaMemcpyAsync(part.data(), dev + ctx->q, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaFreeAsync(dev, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    double num = 0.0, den = 0.0;
    for (int b = 0; b < nb; ++b)
    {
        num += part[2 * b];
        den += part[2 * b + 1];
    }
    if (sums)
    {
        sums[0] = num;
        sums[1] = den;
    }
    // zero reference moment: report the absolute error
    *E = den < 1e-300 ? num : num / den;
    return MRLBM_OK;
}

int mrlbm_set_profiling(mrlbm_ctx* ctx, int on)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    ctx->profiling = on < 0 ? 0 : (on > 2 ? 2 : on);
    return MRLBM_OK;
}

int mrlbm_profile_text(mrlbm_ctx* ctx, char* buf, int cap, int reset)
{
    if (!ctx || !buf || cap <= 0)
        return MRLBM_ERR_CONFIG;
    std::string out;
    for (const auto& kv : ctx->kacc)
        out += kv.first.first + " " + std::to_string(kv.first.second) + " " + std::to_string(kv.second.first) + " " +
               std::to_string(kv.second.second) + "\n";
    const int n = std::min<int>(cap - 1, static_cast<int>(out.size()));
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
    if (reset)
        ctx->kacc.clear();
    return MRLBM_OK;
}

static void drop_graphs(mrlbm_ctx* ctx)
{
    for (auto& gph : ctx->graph)
        if (gph)
        {
            cudaGraphExecDestroy(gph);
            gph = nullptr;
        }
}

static void free_force(mrlbm_ctx* ctx)
{
    cudaFree(ctx->frc);
    cudaFree(ctx->fhist);
    cudaFree(ctx->fhn);
    ctx->frc = nullptr;
    ctx->fhist = nullptr;
    ctx->fhn = nullptr;
    ctx->fcap = 0;
}

// obstacle boxes: per level, the cells whose box can meet the disc's bounding box
// (obstacle_alpha's rejection test) plus two cells of margin, clipped to the level box;
// their alpha values are tabulated once (k_alpha_table), bit-identical to computing
// them per step
static int init_obstacle(mrlbm_ctx* ctx)
{
    long long tot = 0;
    for (int li = 0; li < ctx->nlev; ++li)
    {
        const int m = ctx->J0 + li;
        const double dx = std::ldexp(1.0, -m);
        int lo[2], n[2];
        const int ext[2] = {ctx->geo.nx[li], ctx->geo.ny[li]};
        for (int a = 0; a < 2; ++a)
        {
            const double c0 = ctx->rc.obstacle_center[a] - ctx->rc.obstacle_radius - ctx->rc.origin[a];
            const double c1 = ctx->rc.obstacle_center[a] + ctx->rc.obstacle_radius - ctx->rc.origin[a];
            int a0 = static_cast<int>(std::floor(c0 / dx)) - 2, a1 = static_cast<int>(std::floor(c1 / dx)) + 2;
            a0 = std::max(a0, 0);
            a1 = std::min(a1, ext[a] - 1);
            lo[a] = a0;
            n[a] = std::max(0, a1 - a0 + 1);
        }
        ctx->frc_x0[li] = lo[0];
        ctx->frc_y0[li] = lo[1];
        ctx->frc_nx[li] = n[0];
        ctx->frc_ny[li] = n[1];
        ctx->frc_off[li] = tot;
        tot += static_cast<long long>(n[0]) * n[1];
    }
    ctx->frc_n = tot;
    CU(cudaMalloc(&ctx->alpha_tab, sizeof(double) * std::max(tot, 1LL)));
    for (int li = 0; li < ctx->nlev; ++li)
        if (ctx->frc_nx[li] > 0 && ctx->frc_ny[li] > 0)
            k_alpha_table<<<grid_for(ctx, (long long)ctx->frc_nx[li] * ctx->frc_ny[li]), 256, 0, ctx->stream>>>(
                ctx->sch, ctx->J0 + li, ctx->frc_x0[li], ctx->frc_y0[li], ctx->frc_nx[li], ctx->frc_ny[li],
                ctx->alpha_tab + ctx->frc_off[li]);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    return MRLBM_OK;
}

int mrlbm_set_force_tracking(mrlbm_ctx* ctx, int capacity_steps)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return set_err(ctx, MRLBM_ERR_CONFIG, "force tracking needs the D2Q9 obstacle configuration");
    if (capacity_steps < 0)
        return set_err(ctx, MRLBM_ERR_CONFIG, "force tracking: negative capacity");
    if (capacity_steps > 0 && !(ctx->rc.obstacle == 1 && ctx->D == 2 && ctx->sc.equilibrium == MRLBM_EQ_NS_D2Q9))
        return set_err(ctx, MRLBM_ERR_CONFIG, "force tracking needs the D2Q9 obstacle configuration (obstacle = 1)");
    CU(cudaStreamSynchronize(ctx->stream));
    drop_graphs(ctx);
    free_force(ctx);
    if (capacity_steps == 0)
        return MRLBM_OK;
    const long long tot = ctx->frc_n;
    CU(cudaMalloc(&ctx->frc, sizeof(double) * 2 * std::max(tot, 1LL)));
    CU(cudaMalloc(&ctx->fhist, sizeof(double) * 2 * capacity_steps));
    CU(cudaMalloc(&ctx->fhn, sizeof(int)));
    CU(cudaMemsetAsync(ctx->fhn, 0, sizeof(int), ctx->stream));
    ctx->fcap = capacity_steps;
    return MRLBM_OK;
}

int mrlbm_force_history(mrlbm_ctx* ctx, double* fx, double* fy, int cap, int* n)
{
    if (!ctx || !n)
        return MRLBM_ERR_CONFIG;
    if (!ctx->frc)
        return set_err(ctx, MRLBM_ERR_STATE, "force history: tracking is off");
    int k = 0;
    CU(cudaMemcpyAsync(&k, ctx->fhn, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    const int kk = std::min(std::min(k, ctx->fcap), cap);
    std::vector<double> h(2 * static_cast<size_t>(std::max(kk, 0)));
    if (kk > 0)
    {
        CU(cudaMemcpyAsync(h.data(), ctx->fhist, sizeof(double) * 2 * kk, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    for (int i = 0; i < kk; ++i)
    {
        fx[i] = h[2 * i];
        fy[i] = h[2 * i + 1];
    }
    *n = k;
    if (k > ctx->fcap)
        return set_err(ctx, MRLBM_ERR_CAPACITY, "force history: more steps than the tracking capacity");
    return MRLBM_OK;
}

int mrlbm_tie_log(mrlbm_ctx* ctx, mrlbm_tie_record* out, int cap, int64_t* n, int reset)
{
    if (!ctx || !n || cap < 0)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_tie_log(ctx->e3, out, cap, n, reset);
    int total = 0;
    CU(cudaMemcpyAsync(&total, ctx->tie_n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *n = total;
    const int stored = std::min(total, ctx->tie_cap);
    if (out && cap > 0 && stored > 0)
    {
        std::vector<mrlbm_tie_record> r(stored);
        CU(cudaMemcpy(r.data(), ctx->ties, sizeof(mrlbm_tie_record) * stored, cudaMemcpyDeviceToHost));
        // the device appends in arrival order: sort into (step, level, cell, which)
        std::sort(r.begin(), r.end(), [](const mrlbm_tie_record& a, const mrlbm_tie_record& b) {
            if (a.step != b.step) return a.step < b.step;
            if (a.level != b.level) return a.level < b.level;
            for (int k = 0; k < 3; ++k)
                if (a.cell[k] != b.cell[k]) return a.cell[k] < b.cell[k];
            return a.which < b.which;
        });
        std::memcpy(out, r.data(), sizeof(mrlbm_tie_record) * std::min(cap, stored));
    }
    if (reset)
        CU(cudaMemsetAsync(ctx->tie_n, 0, sizeof(int), ctx->stream));
    return total > ctx->tie_cap ? set_err(ctx, MRLBM_ERR_CAPACITY, "tie log overflow: " + std::to_string(total) +
                                                                      " records, capacity " + std::to_string(ctx->tie_cap))
                                : MRLBM_OK;
}

int mrlbm_set_graph(mrlbm_ctx* ctx, int on)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    ctx->use_graph = on != 0;
    return MRLBM_OK;
}

void* mrlbm_stream_handle(mrlbm_ctx* ctx)
{
    if (ctx && ctx->e3)
        return mrlbm_b200::e3_stream(ctx->e3);
    return ctx ? static_cast<void*>(ctx->stream) : nullptr;
}

int mrlbm_synchronize(mrlbm_ctx* ctx)
{
    if (!ctx)
        return MRLBM_ERR_CONFIG;
    if (ctx->e3)
        return mrlbm_b200::e3_synchronize(ctx->e3);
    CU(cudaStreamSynchronize(ctx->stream));
    return MRLBM_OK;
}

const char* mrlbm_last_error(const mrlbm_ctx* ctx)
{
    if (ctx && ctx->e3 && ctx->err_msg.empty())
        return mrlbm_b200::e3_last_error(ctx->e3);
    return ctx ? ctx->err_msg.c_str() : "null context";
}

void mrlbm_destroy(mrlbm_ctx* ctx)
{
    if (!ctx)
        return;
    if (ctx->e3)
    {
        mrlbm_b200::e3_destroy(ctx->e3);
        delete ctx;
        return;
    }
    if (ctx->stream)
        cudaStreamSynchronize(ctx->stream);
    for (auto& gph : ctx->graph)
        if (gph)
            cudaGraphExecDestroy(gph);
    free_force(ctx);
    cudaFree(ctx->alpha_tab);
    cudaFree(ctx->rdcnt);
    for (int v = 0; v < 2; ++v)
    {
        cudaFree(ctx->cnt[v]);
        for (int li = 0; li < kL; ++li)
        {
            cudaFree(ctx->kind2[v][li]);
            cudaFree(ctx->cells[v][li]);
            cudaFree(ctx->skind[v][li]);
            cudaFree(ctx->F[v][li]);
        }
    }
    for (int li = 0; li < kL; ++li)
    {
        cudaFree(ctx->ld_idx[li]);
        cudaFree(ctx->ld_lin[li]);
        cudaFree(ctx->rn[li]);
        cudaFree(ctx->keep[li]);
        cudaFree(ctx->fbmd[li]);
        cudaFree(ctx->fbdd[li]);
        cudaFree(ctx->tiles[li]);
    }
    cudaFree(ctx->sch);
    cudaFree(ctx->dirty_d);
    cudaFree(ctx->ld_bad);
    cudaFree(ctx->err);
    cudaFree(ctx->fbc);
    cudaFree(ctx->fbs);
    cudaFree(ctx->fbl);
    cudaFree(ctx->fbm);
    cudaFree(ctx->fbdm);
    cudaFree(ctx->upd);
    cudaFree(ctx->ties);
    cudaFree(ctx->tie_n);
    cudaFree(ctx->step_no);
    cudaFree(ctx->tidx);
    cudaFree(ctx->toff);
    cudaFree(ctx->tw);
    cudaFree(ctx->tdep);
    cudaFree(ctx->tpidx);
    cudaFree(ctx->tpar);
    cudaFree(ctx->udep);
    cudaFree(ctx->guidx);
    cudaFree(ctx->guoff);
    cudaFree(ctx->tu);
    cudaFree(ctx->upidx);
    cudaFree(ctx->upar);
    cudaFree(ctx->etad);
    cudaFree(ctx->pmaskd);
    cudaFree(ctx->umaskd);
    for (int i = 0; i < 5; ++i)
    {
        if (ctx->side[i])
            cudaStreamDestroy(ctx->side[i]);
        if (ctx->ev_join[i])
            cudaEventDestroy(ctx->ev_join[i]);
    }
    if (ctx->ev_fork)
        cudaEventDestroy(ctx->ev_fork);
    for (auto& e : ctx->ev)
        if (e)
            cudaEventDestroy(e);
    for (auto& e : ctx->kev)
        cudaEventDestroy(e);
    if (ctx->stream)
        cudaStreamDestroy(ctx->stream);
    delete ctx;
}

} // extern "C"
