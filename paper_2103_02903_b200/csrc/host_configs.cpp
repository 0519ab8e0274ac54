// host_configs.cpp — host-side builders of the product (no CUDA here):
//   * SchemeSpec / RunConfig for the five BASELINE configurations (SPEC.md:372-416
//     for the paper schemes, DESIGN.md Decisions for the three schemes that exist
//     in neither SPEC nor PAPER),
//   * M^-1 by Gauss-Jordan with partial pivoting, same elimination order as the
//     reference DenseMatrix::inverse (dense_matrix.hpp:58-113) so M^-1 is bit-equal,
//   * the flattened reconstruction tables in a "push"
//     (adjoint) formulation with exact dyadic arithmetic,
//   * initial data at equilibrium on the full finest mesh.
#include "mrlbm_internal.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <vector>

namespace mrlbm_b200 {

using I128 = __int128;

bool gauss_jordan_inverse(int n, const double* a_in, double* out)
{
    std::vector<double> a(a_in, a_in + n * n), inv(n * n, 0.0);
    for (int i = 0; i < n; ++i)
        inv[i * n + i] = 1.0;
    for (int col = 0; col < n; ++col)
    {
        int piv = col;
        double best = std::fabs(a[col * n + col]);
        for (int r = col + 1; r < n; ++r)
        {
            const double v = std::fabs(a[r * n + col]);
            if (v > best)
            {
                best = v;
                piv = r;
            }
        }
        if (best == 0.0)
            return false;
        if (piv != col)
            for (int c = 0; c < n; ++c)
            {
                std::swap(a[piv * n + c], a[col * n + c]);
                std::swap(inv[piv * n + c], inv[col * n + c]);
            }
        const double d = 1.0 / a[col * n + col];
        for (int j = 0; j < n; ++j)
        {
            a[col * n + j] *= d;
            inv[col * n + j] *= d;
        }
        for (int r = 0; r < n; ++r)
        {
            if (r == col)
                continue;
            const double f = a[r * n + col];
            if (f == 0.0)
                continue;
            for (int j = 0; j < n; ++j)
            {
                a[r * n + j] -= f * a[col * n + j];
                inv[r * n + j] -= f * inv[col * n + j];
            }
        }
    }
    std::memcpy(out, inv.data(), sizeof(double) * n * n);
    return true;
}

// Prediction weights for gamma = 1 as numerators: W[delta][o] / 8 (1D) or / 64 (2D).
// 1D: P(delta) = f0 + (-1)^delta * c1 * (f+ - f-), c1 = -1/8   (prediction.hpp:149-152)
// 2D: f0 + s0 qx + s1 qy - s0 s1 qxy                            (prediction.hpp:153-159)
static void prediction_numerators(int d, int delta_code, long long* W)
{
    if (d == 1)
    {
        const long long s = (delta_code & 1) ? -1 : 1;
        W[0] = s;  // offset -1 : -(c1) * s * 8 = +s
        W[1] = 8;  // offset 0
        W[2] = -s; // offset +1
        return;
    }
    const long long s0 = ((delta_code >> 1) & 1) ? -1 : 1; // x (axis 0)
    const long long s1 = (delta_code & 1) ? -1 : 1;        // y (axis 1)
    for (int o = 0; o < 9; ++o)
        W[o] = 0;
    auto at = [&](int ox, int oy) -> long long& { return W[(ox + 1) * 3 + (oy + 1)]; };
    at(0, 0) += 64;
    // s0 * qx, qx = -1/8 (f(1,0) - f(-1,0))
    at(1, 0) += -8 * s0;
    at(-1, 0) += 8 * s0;
    at(0, 1) += -8 * s1;
    at(0, -1) += 8 * s1;
    // - s0 s1 qxy, qxy = 1/64 (f(1,1) - f(-1,1) - f(1,-1) + f(-1,-1))
    const long long t = -s0 * s1;
    at(1, 1) += t;
    at(-1, 1) += -t;
    at(1, -1) += -t;
    at(-1, -1) += t;
}

// Push formulation: start from the indicator of the E (side 0) or A (side 1)
// finest cells of a leaf at gap g and push weights down one level at a time
// through the adjoint of the prediction operator.
int build_stream_table(int d, int g, const int32_t* eta, int side, std::vector<TableEntry>& out, TableSets* sets)
{
    out.clear();
    if (d < 1 || d > 2 || g < 0 || g > 14)
        return MRLBM_ERR_CONFIG;
    const long long n = 1LL << g;
    const int shift = (d == 1) ? 3 : 6;
    // finest cells, coordinates relative to the leaf's finest origin
    std::map<std::pair<long long, long long>, I128> cur;
    const long long ylo = (d == 2) ? -1 : 0, yhi = (d == 2) ? n + 1 : 1;
    auto inB = [&](long long x, long long y) { return x >= 0 && x < n && (d == 1 || (y >= 0 && y < n)); };
    for (long long x = -1; x < n + 1; ++x)
        for (long long y = ylo; y < yhi; ++y)
        {
            const long long xe = x + eta[0], ye = (d == 2) ? y + eta[1] : y;
            const bool member = side == 0 ? (inB(xe, ye) && !inB(x, y)) : (inB(x, y) && !inB(xe, ye));
            if (member)
                cur[{x, y}] = 1;
        }
    long long W[4][9];
    for (int s = 0; s < (1 << d); ++s)
        prediction_numerators(d, s, W[s]);
    if (sets)
    {
        // support propagation without cancellation: every cell the recursion touches
        std::map<std::pair<long long, long long>, int> touched;
        for (const auto& kv : cur)
            touched[kv.first] = 1;
        std::map<std::pair<long long, long long>, int> par;
        for (int lvl = g; lvl > 0; --lvl)
        {
            std::map<std::pair<long long, long long>, int> nxt;
            for (const auto& kv : touched)
            {
                const long long px = kv.first.first >> 1, py = (d == 2) ? (kv.first.second >> 1) : 0;
                if (lvl == 1)
                    par[{px, py}] = 1; // parent (level l) of a touched level-(l+1) cell
                for (int ox = -1; ox <= 1; ++ox)
                    for (int oy = (d == 2 ? -1 : 0); oy <= (d == 2 ? 1 : 0); ++oy)
                        nxt[{px + ox, py + oy}] = 1;
            }
            touched.swap(nxt);
        }
        sets->dep_lo[0] = sets->dep_lo[1] = 1 << 30;
        sets->dep_hi[0] = sets->dep_hi[1] = -(1 << 30);
        for (const auto& kv : touched)
        {
            const int x = static_cast<int>(kv.first.first), y = static_cast<int>(kv.first.second);
            sets->dep_lo[0] = std::min(sets->dep_lo[0], x);
            sets->dep_hi[0] = std::max(sets->dep_hi[0], x);
            sets->dep_lo[1] = std::min(sets->dep_lo[1], y);
            sets->dep_hi[1] = std::max(sets->dep_hi[1], y);
        }
        if (touched.empty())
            sets->dep_lo[0] = sets->dep_lo[1] = sets->dep_hi[0] = sets->dep_hi[1] = 0;
        sets->par.clear();
        for (const auto& kv : par)
            sets->par.emplace_back(static_cast<int>(kv.first.first), static_cast<int>(kv.first.second));
    }
    for (int lvl = g; lvl > 0; --lvl)
    {
        std::map<std::pair<long long, long long>, I128> nxt;
        for (const auto& [c, w] : cur)
        {
            if (w == 0)
                continue;
            const long long px = c.first >> 1, py = (d == 2) ? (c.second >> 1) : 0;
            const int dx = static_cast<int>(c.first - 2 * px);
            const int dy = (d == 2) ? static_cast<int>(c.second - 2 * py) : 0;
            const int code = (d == 1) ? dx : (dx << 1) | dy;
            if (d == 1)
            {
                for (int o = -1; o <= 1; ++o)
                    nxt[{px + o, 0}] += w * W[code][o + 1];
            }
            else
            {
                for (int ox = -1; ox <= 1; ++ox)
                    for (int oy = -1; oy <= 1; ++oy)
                    {
                        const long long wn = W[code][(ox + 1) * 3 + (oy + 1)];
                        if (wn != 0)
                            nxt[{px + ox, py + oy}] += w * wn;
                    }
            }
        }
        cur.swap(nxt);
    }
    for (const auto& [c, w] : cur)
    {
        if (w == 0)
            continue;
        TableEntry e{};
        e.off[0] = static_cast<int>(c.first);
        e.off[1] = static_cast<int>(c.second);
        // round-to-nearest of the exact dyadic rational (int128 -> double is
        // correctly rounded; the power-of-two scaling is exact).  Weights are
        // exact up to gap 9; diagonal velocities need 54+ bits from gap 10 on.
        const double v = std::ldexp(static_cast<double>(w), -shift * g);
        if (std::abs(e.off[0]) > 2 || std::abs(e.off[1]) > 2)
            return MRLBM_ERR_CAPACITY; // outside the 5^d neighbourhood
        e.w = v;
        out.push_back(e);
    }
    return MRLBM_OK; // std::map order == lexicographic (x, y)
}

// 3D push builder (gamma = 1).  Prediction weights as numerators over 512
// (prediction.hpp:160-172 with c = -1/8): centre 512; axis a at sigma e_a:
// -64 s_a sigma; plane (a, b) at (sigma_a, sigma_b): -8 s_a s_b sigma_a sigma_b (the
// reference's minus sign on the plane terms); corner: -s_0 s_1 s_2 sigma_0 sigma_1 sigma_2,
// with s_a = +1 for child selector delta_a = 0, -1 for delta_a = 1.
int build_stream_table3(int g, const int32_t* eta, int side, std::vector<TableEntry3>& out, TableSets3* sets)
{
    using Key = std::array<long long, 3>;
    out.clear();
    if (g < 0 || g > 12)
        return MRLBM_ERR_CONFIG;
    const long long n = 1LL << g;
    auto inB = [&](const Key& x) {
        for (int a = 0; a < 3; ++a)
            if (x[a] < 0 || x[a] >= n)
                return false;
        return true;
    };
    std::map<Key, I128> cur;
    // E = (B - eta) \ B, A = B \ (B - eta): candidates are the cells of B - eta (E) or B (A)
    for (long long x = 0; x < n; ++x)
        for (long long y = 0; y < n; ++y)
            for (long long z = 0; z < n; ++z)
            {
                const Key b{x, y, z};
                const Key c = side == 0 ? Key{x - eta[0], y - eta[1], z - eta[2]} : b;
                const Key ce{c[0] + eta[0], c[1] + eta[1], c[2] + eta[2]};
                const bool member = side == 0 ? (inB(ce) && !inB(c)) : (inB(c) && !inB(ce));
                if (member)
                    cur[c] = 1;
            }
    long long W[8][27];
    for (int code = 0; code < 8; ++code)
    {
        const long long s[3] = {(code >> 2) & 1 ? -1 : 1, (code >> 1) & 1 ? -1 : 1, code & 1 ? -1 : 1};
        for (int o = 0; o < 27; ++o)
        {
            const long long sg[3] = {o / 9 - 1, (o / 3) % 3 - 1, o % 3 - 1};
            const int nz = (sg[0] != 0) + (sg[1] != 0) + (sg[2] != 0);
            long long w = 0;
            if (nz == 0)
                w = 512;
            else if (nz == 1)
            {
                for (int a = 0; a < 3; ++a)
                    if (sg[a] != 0)
                        w = -64 * s[a] * sg[a];
            }
            else if (nz == 2)
            {
                w = -8;
                for (int a = 0; a < 3; ++a)
                    if (sg[a] != 0)
                        w *= s[a] * sg[a];
            }
            else
                w = -(s[0] * sg[0]) * (s[1] * sg[1]) * (s[2] * sg[2]);
            W[code][o] = w;
        }
    }
    if (sets)
    {
        std::map<Key, int> touched, par;
        for (const auto& kv : cur)
            touched[kv.first] = 1;
        for (int lvl = g; lvl > 0; --lvl)
        {
            std::map<Key, int> nxt;
            for (const auto& kv : touched)
            {
                const Key p{kv.first[0] >> 1, kv.first[1] >> 1, kv.first[2] >> 1};
                if (lvl == 1)
                    par[p] = 1;
                for (int o = 0; o < 27; ++o)
                    nxt[Key{p[0] + o / 9 - 1, p[1] + (o / 3) % 3 - 1, p[2] + o % 3 - 1}] = 1;
            }
            touched.swap(nxt);
        }
        for (int a = 0; a < 3; ++a)
        {
            sets->dep_lo[a] = touched.empty() ? 0 : (1 << 30);
            sets->dep_hi[a] = touched.empty() ? 0 : -(1 << 30);
        }
        for (const auto& kv : touched)
            for (int a = 0; a < 3; ++a)
            {
                sets->dep_lo[a] = std::min(sets->dep_lo[a], static_cast<int>(kv.first[a]));
                sets->dep_hi[a] = std::max(sets->dep_hi[a], static_cast<int>(kv.first[a]));
            }
        sets->par.clear();
        for (const auto& kv : par)
            sets->par.push_back({static_cast<int>(kv.first[0]), static_cast<int>(kv.first[1]), static_cast<int>(kv.first[2])});
    }
    for (int lvl = g; lvl > 0; --lvl)
    {
        std::map<Key, I128> nxt;
        for (const auto& [c, w] : cur)
        {
            if (w == 0)
                continue;
            const Key p{c[0] >> 1, c[1] >> 1, c[2] >> 1};
            const int code = static_cast<int>(((c[0] - 2 * p[0]) << 2) | ((c[1] - 2 * p[1]) << 1) | (c[2] - 2 * p[2]));
            for (int o = 0; o < 27; ++o)
                nxt[Key{p[0] + o / 9 - 1, p[1] + (o / 3) % 3 - 1, p[2] + o % 3 - 1}] += w * W[code][o];
        }
        cur.swap(nxt);
    }
    for (const auto& [c, w] : cur)
    {
        if (w == 0)
            continue;
        TableEntry3 e{};
        for (int a = 0; a < 3; ++a)
            e.off[a] = static_cast<int>(c[a]);
        e.w = std::ldexp(static_cast<double>(w), -9 * g); // nearest double to the exact dyadic (D.12)
        out.push_back(e);
    }
    return MRLBM_OK; // std::map order == lexicographic (x, y, z)
}

} // namespace mrlbm_b200

using namespace mrlbm_b200;

namespace {

void set_M_d2q4(double* M, int q, int base, double lam)
{
    const double r[4][4] = {{1, 1, 1, 1}, {lam, 0, -lam, 0}, {0, lam, 0, -lam}, {lam * lam, -lam * lam, lam * lam, -lam * lam}};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            M[(base + i) * q + base + j] = r[i][j];
}

const int32_t kD2Q4[4][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};

double euler_energy(double rho, double u, double v, double p, double gam)
{
    return p / (gam - 1.0) + 0.5 * rho * (u * u + v * v);
}

// splitmix64 -> uniform in [-1, 1): the seeded perturbation of config 5 (Decision D.16)
double splitmix_unit(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    x = x ^ (x >> 31);
    return static_cast<double>(x >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

} // namespace

extern "C" {

int mrlbm_stream_table(int d, int gap, const int32_t eta[3], int side, int cap, int32_t* offsets, double* weights, int* n)
{
    if (d == 3)
    {
        std::vector<TableEntry3> t3;
        const int st3 = build_stream_table3(gap, eta, side, t3, nullptr);
        if (st3 != MRLBM_OK)
            return st3;
        if (static_cast<int>(t3.size()) > cap)
            return MRLBM_ERR_CAPACITY;
        for (size_t i = 0; i < t3.size(); ++i)
        {
            for (int a = 0; a < 3; ++a)
                offsets[i * 3 + a] = t3[i].off[a];
            weights[i] = t3[i].w;
        }
        *n = static_cast<int>(t3.size());
        return MRLBM_OK;
    }
    std::vector<TableEntry> t;
    const int st = build_stream_table(d, gap, eta, side, t);
    if (st != MRLBM_OK)
        return st;
    if (static_cast<int>(t.size()) > cap)
        return MRLBM_ERR_CAPACITY;
    for (size_t i = 0; i < t.size(); ++i)
    {
        for (int a = 0; a < d; ++a)
            offsets[i * d + a] = t[i].off[a];
        weights[i] = t[i].w;
    }
    *n = static_cast<int>(t.size());
    return MRLBM_OK;
}

// equilibrium populations M^-1 m^eq for host-side initial data
static void host_feq(const mrlbm_scheme_spec* sc, const double* cons, double* f)
{
    const int q = sc->q;
    double meq[MRLBM_MAX_Q] = {0};
    switch (sc->equilibrium)
    {
        case MRLBM_EQ_BURGERS_D1Q2:
            meq[0] = cons[0];
            meq[1] = 0.5 * cons[0] * cons[0];
            break;
        case MRLBM_EQ_EULER_D1Q3X3:
        {
            const double gam = sc->eq_params[0], lam2 = sc->lambda * sc->lambda;
            const double rho = cons[0], qq = cons[1], E = cons[2];
            const double u = qq / rho;
            const double p = (gam - 1.0) * (E - 0.5 * rho * u * u);
            const double F[3] = {qq, qq * u + p, u * (E + p)};
            for (int i = 0; i < 3; ++i)
            {
                meq[3 * i] = cons[i];
                meq[3 * i + 1] = F[i];
                meq[3 * i + 2] = lam2 * cons[i];
            }
            break;
        }
        case MRLBM_EQ_ADVECTION_D2Q4:
            meq[0] = cons[0];
            meq[1] = sc->eq_params[0] * cons[0];
            meq[2] = sc->eq_params[1] * cons[0];
            meq[3] = 0.0;
            break;
        case MRLBM_EQ_EULER_D2Q4X4:
        {
            const double gam = sc->eq_params[0];
            const double rho = cons[0], qx = cons[1], qy = cons[2], E = cons[3];
            const double u = qx / rho, v = qy / rho;
            const double p = (gam - 1.0) * (E - 0.5 * rho * (u * u + v * v));
            const double Fx[4] = {qx, qx * u + p, qx * v, u * (E + p)};
            const double Fy[4] = {qy, qy * u, qy * v + p, v * (E + p)};
            for (int i = 0; i < 4; ++i)
            {
                meq[4 * i] = cons[i];
                meq[4 * i + 1] = Fx[i];
                meq[4 * i + 2] = Fy[i];
                meq[4 * i + 3] = 0.0;
            }
            break;
        }
        case MRLBM_EQ_NS_D2Q9:
        {
            const double cs2 = sc->eq_params[0];
            const double rho = cons[0], qx = cons[1], qy = cons[2];
            const double q2 = qx * qx + qy * qy;
            meq[0] = rho;
            meq[1] = qx;
            meq[2] = qy;
            meq[3] = 3.0 * (-2.0 * cs2 * rho + q2 / rho);
            meq[4] = -3.0 * cs2 * qx;
            meq[5] = -3.0 * cs2 * qy;
            meq[6] = 9.0 * (cs2 * cs2 * rho - cs2 * q2 / rho);
            meq[7] = (qx * qx - qy * qy) / rho;
            meq[8] = qx * qy / rho;
            break;
        }
        case MRLBM_EQ_ADVECTION_D3Q6:
            meq[0] = cons[0];
            meq[1] = sc->eq_params[0] * cons[0];
            meq[2] = sc->eq_params[1] * cons[0];
            meq[3] = sc->eq_params[2] * cons[0];
            break;
    }
    for (int i = 0; i < q; ++i)
    {
        double acc = 0.0;
        for (int j = 0; j < q; ++j)
            acc += sc->Minv[i * q + j] * meq[j];
        f[i] = acc;
    }
}

int mrlbm_stream_table_sets(int d, int gap, const int32_t eta[3], int side, int cap, int32_t* dep_box,
                            int32_t* par_offsets, int* npar)
{
    std::vector<TableEntry> t;
    TableSets ts{};
    const int st = build_stream_table(d, gap, eta, side, t, &ts);
    if (st != MRLBM_OK)
        return st;
    if (static_cast<int>(ts.par.size()) > cap)
        return MRLBM_ERR_CAPACITY;
    dep_box[0] = ts.dep_lo[0];
    dep_box[1] = ts.dep_hi[0];
    dep_box[2] = ts.dep_lo[1];
    dep_box[3] = ts.dep_hi[1];
    for (size_t i = 0; i < ts.par.size(); ++i)
    {
        par_offsets[i * d] = ts.par[i].first;
        if (d == 2)
            par_offsets[i * d + 1] = ts.par[i].second;
    }
    *npar = static_cast<int>(ts.par.size());
    return MRLBM_OK;
}

int mrlbm_build_config(int id, int jmax_override, double eps_override, mrlbm_scheme_spec* sc, mrlbm_run_config* rc)
{
    std::memset(sc, 0, sizeof(*sc));
    std::memset(rc, 0, sizeof(*rc));
    rc->gamma = 1;
    rc->graduation = 1;
    rc->obstacle_subsamples = 16;
    sc->nblocks = 1;
    switch (id)
    {
        case 1: // D1Q2 Burgers on [-3,3], levels 2..10 (Decisions D.2, D.18)
        {
            sc->d = 1;
            sc->q = 2;
            sc->equilibrium = MRLBM_EQ_BURGERS_D1Q2;
            sc->lambda = 1.0;
            sc->eta[0][0] = 1;
            sc->eta[1][0] = -1;
            const double lam = sc->lambda;
            const double M[4] = {1, 1, lam, -lam};
            std::memcpy(sc->M, M, sizeof(M));
            sc->s[0] = 0.0;
            sc->s[1] = 1.5;
            rc->j_min = 2;
            rc->j_max = 10;
            rc->base_cells[0] = 4 * 6;
            rc->origin[0] = -3.0;
            rc->epsilon = 1e-4;
            rc->mu = 0;
            rc->bc_kind[0] = rc->bc_kind[1] = MRLBM_BC_COPY;
            break;
        }
        case 2: // three coupled D1Q3 (rho, rho u, E), Lax data (Decision D.19)
        {
            sc->d = 1;
            sc->q = 9;
            sc->nblocks = 3;
            sc->equilibrium = MRLBM_EQ_EULER_D1Q3X3;
            sc->lambda = 3.0;
            sc->eq_params[0] = 1.4;
            const double lam = sc->lambda;
            for (int b = 0; b < 3; ++b)
            {
                const int base = 3 * b;
                sc->eta[base + 0][0] = 0;
                sc->eta[base + 1][0] = 1;
                sc->eta[base + 2][0] = -1;
                const double r[3][3] = {{1, 1, 1}, {0, lam, -lam}, {0, lam * lam, lam * lam}};
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        sc->M[(base + i) * 9 + base + j] = r[i][j];
                sc->s[base + 0] = 0.0;
                sc->s[base + 1] = 1.9;
                sc->s[base + 2] = 1.9;
            }
            rc->j_min = 2;
            rc->j_max = 14;
            rc->base_cells[0] = 4;
            rc->epsilon = 1e-4;
            rc->mu = 0;
            rc->bc_kind[0] = rc->bc_kind[1] = MRLBM_BC_COPY;
            break;
        }
        case 3: // D2Q4 advection, periodic (Decision D.20)
        {
            sc->d = 2;
            sc->q = 4;
            sc->equilibrium = MRLBM_EQ_ADVECTION_D2Q4;
            sc->lambda = 1.0;
            sc->eq_params[0] = 1.0; // a
            sc->eq_params[1] = 1.0; // b
            for (int h = 0; h < 4; ++h)
            {
                sc->eta[h][0] = kD2Q4[h][0];
                sc->eta[h][1] = kD2Q4[h][1];
            }
            set_M_d2q4(sc->M, 4, 0, sc->lambda);
            sc->s[0] = 0.0;
            sc->s[1] = sc->s[2] = sc->s[3] = 1.9;
            rc->j_min = 2;
            rc->j_max = 9;
            rc->base_cells[0] = rc->base_cells[1] = 4;
            rc->epsilon = 1e-4;
            rc->mu = 0;
            for (int f = 0; f < 4; ++f)
                rc->bc_kind[f] = MRLBM_BC_PERIODIC;
            break;
        }
        case 4: // D2Q4^4 Euler, four-quadrant Riemann problem (Decision D.21)
        {
            sc->d = 2;
            sc->q = 16;
            sc->nblocks = 4;
            sc->equilibrium = MRLBM_EQ_EULER_D2Q4X4;
            sc->lambda = 4.0;
            sc->eq_params[0] = 1.4;
            for (int b = 0; b < 4; ++b)
            {
                for (int h = 0; h < 4; ++h)
                {
                    sc->eta[4 * b + h][0] = kD2Q4[h][0];
                    sc->eta[4 * b + h][1] = kD2Q4[h][1];
                }
                set_M_d2q4(sc->M, 16, 4 * b, sc->lambda);
                sc->s[4 * b] = 0.0;
                sc->s[4 * b + 1] = sc->s[4 * b + 2] = sc->s[4 * b + 3] = 1.9;
            }
            rc->j_min = 2;
            rc->j_max = 11;
            rc->base_cells[0] = rc->base_cells[1] = 4;
            rc->epsilon = 1e-3;
            rc->mu = 0;
            for (int f = 0; f < 4; ++f)
                rc->bc_kind[f] = MRLBM_BC_COPY;
            break;
        }
        case 5: // D2Q9 Navier-Stokes past a cylinder
        {
            sc->d = 2;
            sc->q = 9;
            sc->equilibrium = MRLBM_EQ_NS_D2Q9;
            sc->lambda = 1.0;
            const double lam = sc->lambda;
            const int32_t e9[9][2] = {{0, 0}, {1, 0}, {0, 1}, {-1, 0}, {0, -1}, {1, 1}, {-1, 1}, {-1, -1}, {1, -1}};
            for (int h = 0; h < 9; ++h)
            {
                sc->eta[h][0] = e9[h][0];
                sc->eta[h][1] = e9[h][1];
            }
            const double l2 = lam * lam, l3 = l2 * lam, l4 = l2 * l2;
            const double M[9][9] = {
                {1, 1, 1, 1, 1, 1, 1, 1, 1},
                {0, lam, 0, -lam, 0, lam, -lam, -lam, lam},
                {0, 0, lam, 0, -lam, lam, lam, -lam, -lam},
                {-4 * l2, -l2, -l2, -l2, -l2, 2 * l2, 2 * l2, 2 * l2, 2 * l2},
                {0, -2 * l3, 0, 2 * l3, 0, l3, -l3, -l3, l3},
                {0, 0, -2 * l3, 0, 2 * l3, l3, l3, -l3, -l3},
                {4 * l4, -2 * l4, -2 * l4, -2 * l4, -2 * l4, l4, l4, l4, l4},
                {0, l2, -l2, l2, -l2, 0, 0, 0, 0},
                {0, 0, 0, 0, 0, l2, -l2, l2, -l2}};
            for (int i = 0; i < 9; ++i)
                for (int j = 0; j < 9; ++j)
                    sc->M[i * 9 + j] = M[i][j];
            const double cs2 = l2 / 3.0;
            sc->eq_params[0] = cs2;
            sc->eq_params[1] = 0.0; // |q|^2/rho variant (Decision D.17)
            rc->j_min = 2;
            rc->j_max = 12;
            const double rho0 = 1.0, u0 = 0.05, Re = 1200.0, radius = 0.0625;
            const double L = 2.0 * radius;
            const double mu_visc = rho0 * u0 * L / Re;
            const double dt = std::ldexp(1.0, -rc->j_max) / lam;
            const double s2 = 1.0 / (0.5 + mu_visc / (cs2 * dt * rho0));
            const double s1 = 1.5; // Decision D.17 (PAPER.md:1330 leaves it free)
            const double S[9] = {0, 0, 0, s1, s1, s1, s1, s2, s2};
            std::memcpy(sc->s, S, sizeof(S));
            rc->base_cells[0] = 8;
            rc->base_cells[1] = 4;
            rc->epsilon = 1e-4;
            rc->mu = 1;
            rc->bc_kind[0] = MRLBM_BC_VELOCITY_BOUNCE_BACK; // inlet
            rc->bc_kind[1] = MRLBM_BC_COPY;                 // outlet
            rc->bc_kind[2] = MRLBM_BC_VELOCITY_BOUNCE_BACK; // bottom
            rc->bc_kind[3] = MRLBM_BC_VELOCITY_BOUNCE_BACK; // top
            const double w9[9] = {4.0 / 9, 1.0 / 9, 1.0 / 9, 1.0 / 9, 1.0 / 9, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36};
            for (int f = 0; f < 4; ++f)
                for (int h = 0; h < 9; ++h)
                {
                    // Ladd moving-wall term 2 w_h rho0 (xi_h . u_w) / c_s^2, u_w = (u0, 0)
                    const double xi_u = lam * e9[h][0] * u0;
                    rc->bc_add[f][h] = (f == 1) ? 0.0 : 2.0 * w9[h] * rho0 * xi_u / cs2;
                }
            rc->obstacle = 1;
            rc->obstacle_center[0] = 0.3125;
            rc->obstacle_center[1] = 0.5;
            rc->obstacle_radius = radius;
            break;
        }
        case 6: // D3Q6 advection of the indicator of a sphere (D.28)
        {
            sc->d = 3;
            sc->q = 6;
            sc->equilibrium = MRLBM_EQ_ADVECTION_D3Q6;
            sc->lambda = 1.0;
            const double lam = sc->lambda, l2 = lam * lam;
            const int32_t e6[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
            for (int h = 0; h < 6; ++h)
                for (int a = 0; a < 3; ++a)
                    sc->eta[h][a] = e6[h][a];
            const double M[6][6] = {{1, 1, 1, 1, 1, 1},       {lam, -lam, 0, 0, 0, 0}, {0, 0, lam, -lam, 0, 0},
                                    {0, 0, 0, 0, lam, -lam}, {l2, l2, -l2, -l2, 0, 0}, {l2, l2, 0, 0, -l2, -l2}};
            for (int i = 0; i < 6; ++i)
                for (int j = 0; j < 6; ++j)
                    sc->M[i * 6 + j] = M[i][j] + 0.0;
            const double S[6] = {0, 1.4, 1.4, 1.4, 1.0, 1.0}; // s1 = 1.4, s2 = 1
            std::memcpy(sc->s, S, sizeof(S));
            // V (D.28): inside |V_a| <= lambda / 3, where the equilibrium populations u (1/6 +- V_a / (2 lambda))
            // stay non-negative; V = 1/2 was measured unstable (|u| -> 1e53 in 200 steps)
            sc->eq_params[0] = sc->eq_params[1] = sc->eq_params[2] = 0.25;
            rc->j_min = 1;
            rc->j_max = 8;
            rc->epsilon = 1e-3;
            rc->mu = 2;
            for (int a = 0; a < 3; ++a)
            {
                rc->base_cells[a] = 2;     // unit cube: 2^l cells per axis at level l
                rc->origin[a] = -0.375;    // [-3/8, 5/8]^3: the sphere stays inside until T = 0.78125
            }
            for (int f = 0; f < 6; ++f)
                rc->bc_kind[f] = MRLBM_BC_COPY;
            break;
        }
        default:
            return MRLBM_ERR_CONFIG;
    }
    if (jmax_override > 0)
    {
        if (jmax_override <= rc->j_min)
            return MRLBM_ERR_CONFIG;
        rc->j_max = jmax_override;
        if (id == 5)
        { // s2 depends on dt = 2^-J / lambda
            const double cs2 = sc->eq_params[0];
            const double mu_visc = 1.0 * 0.05 * 0.125 / 1200.0;
            const double dt = std::ldexp(1.0, -rc->j_max) / sc->lambda;
            const double s2 = 1.0 / (0.5 + mu_visc / (cs2 * dt * 1.0));
            sc->s[7] = sc->s[8] = s2;
        }
    }
    if (eps_override >= 0.0)
        rc->epsilon = eps_override;
    if (!gauss_jordan_inverse(sc->q, sc->M, sc->Minv))
        return MRLBM_ERR_CONFIG;
    // compact the q x q inverse (the descriptor stores row-major q x q in the first q*q slots)
    if (id == 5)
    {
        const double cons[3] = {1.0, 0.0, 0.0}; // rho0, u = 0
        host_feq(sc, cons, rc->obstacle_feq);
    }
    return MRLBM_OK;
}

int64_t mrlbm_config_steps(int id, const mrlbm_run_config* rc)
{
    // N = ceil(T / dt), dt = 2^-J / lambda  (Decision D.11)
    const int J = rc->j_max;
    switch (id)
    {
        case 1: return static_cast<int64_t>(std::ceil(2.0 * std::ldexp(1.0, J) / 1.0));
        case 2: return static_cast<int64_t>(std::ceil(0.14 * 3.0 * std::ldexp(1.0, J)));
        case 3: return static_cast<int64_t>(std::ceil(1.0 * 1.0 * std::ldexp(1.0, J)));
        case 4: return static_cast<int64_t>(std::ceil(0.25 * 4.0 * std::ldexp(1.0, J)));
        case 5: return 50000;
        case 6: return static_cast<int64_t>(std::ceil(0.78125 * 1.0 * std::ldexp(1.0, J)));
        default: return -1;
    }
}

int mrlbm_initial_finest(int id, const mrlbm_scheme_spec* sc, const mrlbm_run_config* rc, uint64_t seed, double* f)
{
    const int J = rc->j_max;
    const int64_t nx = rc->base_cells[0] << (J - rc->j_min);
    const int64_t ny = (sc->d >= 2) ? (rc->base_cells[1] << (J - rc->j_min)) : 1;
    const int64_t nz = (sc->d == 3) ? (rc->base_cells[2] << (J - rc->j_min)) : 1;
    const int64_t N = nx * ny * nz;
    const double dx = std::ldexp(1.0, -J);
    const int q = sc->q;
    double fl[MRLBM_MAX_Q];
    for (int64_t ix = 0; ix < nx; ++ix)
        for (int64_t iyz = 0; iyz < ny * nz; ++iyz)
        {
            const int64_t iy = iyz / nz, iz = iyz % nz;
            const int64_t i = ix * ny * nz + iyz;
            const double x = rc->origin[0] + (static_cast<double>(ix) + 0.5) * dx;
            const double y = rc->origin[1] + (static_cast<double>(iy) + 0.5) * dx;
            const double z = rc->origin[2] + (static_cast<double>(iz) + 0.5) * dx;
            double cons[4] = {0, 0, 0, 0};
            switch (id)
            {
                case 1:
                    cons[0] = std::max(0.0, 1.0 - std::fabs(x));
                    break;
                case 2:
                {
                    const double gam = sc->eq_params[0];
                    const bool left = x < 0.5;
                    const double rho = left ? 0.445 : 0.5, u = left ? 0.698 : 0.0, p = left ? 3.528 : 0.571;
                    cons[0] = rho;
                    cons[1] = rho * u;
                    cons[2] = euler_energy(rho, u, 0.0, p, gam);
                    break;
                }
                case 3:
                {
                    const double ddx = x - 0.5, ddy = y - 0.5;
                    cons[0] = (ddx * ddx + ddy * ddy <= 0.2 * 0.2) ? 1.0 : 0.0;
                    break;
                }
                case 4:
                {
                    const double gam = sc->eq_params[0];
                    double rho, u, v, p;
                    if (x > 0.5 && y > 0.5)
                    {
                        rho = 1.5; u = 0.0; v = 0.0; p = 1.5;
                    }
                    else if (x < 0.5 && y > 0.5)
                    {
                        rho = 0.5323; u = 1.206; v = 0.0; p = 0.3;
                    }
                    else if (x < 0.5 && y < 0.5)
                    {
                        rho = 0.138; u = 1.206; v = 1.206; p = 0.029;
                    }
                    else
                    {
                        rho = 0.5323; u = 0.0; v = 1.206; p = 0.3;
                    }
                    cons[0] = rho;
                    cons[1] = rho * u;
                    cons[2] = rho * v;
                    cons[3] = euler_energy(rho, u, v, p, gam);
                    break;
                }
                case 5:
                {
                    const double rho = 1.0;
                    const double v = 1e-3 * splitmix_unit(seed ^ static_cast<uint64_t>(i));
                    cons[0] = rho;
                    cons[1] = 0.0;
                    cons[2] = rho * v;
                    break;
                }
                case 6:
                    cons[0] = (x * x + y * y + z * z <= 0.15 * 0.15) ? 1.0 : 0.0;
                    break;
                default:
                    return MRLBM_ERR_CONFIG;
            }
            host_feq(sc, cons, fl);
            for (int h = 0; h < q; ++h)
                f[h * N + i] = fl[h];
        }
    return MRLBM_OK;
}

// ---- config-5 integral diagnostics ----
int mrlbm_drag_lift(double fx, double fy, double rho0, double u0, double L, double* cd, double* cl)
{
    const double den = rho0 * u0 * u0 * L;
    if (!(den > 0.0) || !cd || !cl)
        return MRLBM_ERR_CONFIG;
    *cd = 2.0 * fx / den;
    *cl = 2.0 * fy / den;
    return MRLBM_OK;
}

int mrlbm_strouhal(const double* cl, int64_t n, int64_t skip, double dt, double u0, double L, double* st, double* df)
{
    if (!cl || !st || skip < 0 || !(dt > 0.0) || !(u0 != 0.0))
        return MRLBM_ERR_CONFIG;
    const int64_t N = n - skip;
    if (N < 8)
        return MRLBM_ERR_CONFIG;
    const double* y = cl + skip;
    // least-squares line a + b t (t = sample index), removed
    double st_ = 0.0, sy = 0.0, stt = 0.0, sty = 0.0;
    for (int64_t i = 0; i < N; ++i)
    {
        const double t = static_cast<double>(i);
        st_ += t;
        sy += y[i];
        stt += t * t;
        sty += t * y[i];
    }
    const double Nd = static_cast<double>(N);
    const double b = (Nd * sty - st_ * sy) / (Nd * stt - st_ * st_);
    const double a = (sy - b * st_) / Nd;
    std::vector<double> w(N);
    double amp = 0.0;
    for (int64_t i = 0; i < N; ++i)
    {
        const double r = y[i] - (a + b * static_cast<double>(i));
        const double hann = 0.5 - 0.5 * std::cos(2.0 * M_PI * static_cast<double>(i) / static_cast<double>(N - 1));
        w[i] = r * hann;
        amp = std::max(amp, std::fabs(r));
    }
    const double scale = std::max(std::fabs(a), std::fabs(b) * Nd);
    if (!(amp > 1e-12 * scale) || amp == 0.0)
        return MRLBM_ERR_NUMERIC; // flat after detrending: no shedding
    // direct DFT power over bins 1 .. N/2
    const int64_t K = N / 2;
    std::vector<double> p(K + 1, 0.0);
    for (int64_t k = 1; k <= K; ++k)
    {
        double re = 0.0, im = 0.0;
        const double wk = 2.0 * M_PI * static_cast<double>(k) / Nd;
        for (int64_t i = 0; i < N; ++i)
        {
            const double ph = wk * static_cast<double>(i);
            re += w[i] * std::cos(ph);
            im -= w[i] * std::sin(ph);
        }
        p[k] = re * re + im * im;
    }
    int64_t kmax = 1;
    for (int64_t k = 2; k <= K; ++k)
        if (p[k] > p[kmax])
            kmax = k;
    double rest = 0.0;
    for (int64_t k = 1; k <= K; ++k)
        if (k != kmax)
            rest += p[k];
    rest /= static_cast<double>(std::max<int64_t>(K - 1, 1));
    if (!(p[kmax] > 4.0 * rest))
        return MRLBM_ERR_NUMERIC; // no dominant peak
    const double freq = static_cast<double>(kmax) / (Nd * dt);
    *st = L * freq / u0;
    if (df)
        *df = 1.0 / (Nd * dt);
    return MRLBM_OK;
}

} // extern "C"
