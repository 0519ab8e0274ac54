// mrlbm_oracle.cpp — CPU ORACLE for the adaptive MR-LBM time step.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2103_02903_b200/)
// links, loads or calls this file; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs do, as the checker.
//
// The reference (/root/reference/proj/core/include/mrlbm) ships the mesh and MR
// primitives only; the step itself exists there as prose (SPEC.md, PAPER.md
// Algorithm 1).  This file restates the step literally on top of the reference
// headers, which it INCLUDES (never copies):
//   CellSet / CellIndex  cell_set.hpp:17-394  (mesh sets, slot order)
//   DomainBox, parent    cell.hpp:102-196
//   project, predict     prediction.hpp:51-60, 143-173
//   DenseMatrix          dense_matrix.hpp:42-113 (collision matvec order, inverse)
// Semantics pinned in DESIGN.md §Decisions (SURVEY Appendix A ledger).
//
// PARITY STATUS: the reference ships no golden vectors for the step, so the
// step is "parity unpinned" against upstream output; the primitives it uses
// are the reference's own code, pinned by tests/test_oracle_prims.py.
//
// Build: oracle/Makefile  (g++ -std=c++20 -O2 -ffp-contract=off -include cmath
//        -I/root/reference/proj/core/include -fopenmp)

#include <mrlbm/cell.hpp>
#include <mrlbm/cell_set.hpp>
#include <mrlbm/dense_matrix.hpp>
#include <mrlbm/prediction.hpp>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <mutex>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <omp.h>

#include "../include/mrlbm_gpu.h"

namespace {

using I64 = std::int64_t;
using I128 = __int128;

// exceptions must not cross an OpenMP region: capture the first, rethrow after
struct OmpErr {
    std::exception_ptr ep;
    std::mutex mu;
    template <class Fn>
    void run(Fn&& fn)
    {
        try
        {
            fn();
        }
        catch (...)
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!ep)
                ep = std::current_exception();
        }
    }
    void rethrow()
    {
        if (ep)
            std::rethrow_exception(ep);
    }
};

// ---------------------------------------------------------------------------
// Flattened reconstruction tables.
// Pull formulation: memoised recursion rec(m, c) over an infinite uniform
// level-l neighbourhood, each rec a linear form over level-l offsets with exact
// dyadic coefficients (numerators over 8^depth in 1D, 64^depth in 2D).  The
// one-hot prediction weights come from calling the reference predict<D>
// (prediction.hpp:143-173), so the minus cross-term convention is the
// reference's.
// ---------------------------------------------------------------------------
// 3^D prediction stencil, entries in lexicographic order (axis 0 slowest):
// offset of entry o along axis a, in {-1, 0, 1}
template <int D>
constexpr int kStencil = (D == 1 ? 3 : (D == 2 ? 9 : 27));

template <int D>
inline int stencil_off(int o, int a)
{
    int div = 1;
    for (int i = D - 1; i > a; --i)
        div *= 3;
    return (o / div) % 3 - 1;
}

template <int D>
struct TableBuilder {
    // W[delta][o] numerators (denominator 8 for D=1, 64 for D=2, 512 for D=3)
    std::array<std::array<I64, kStencil<D>>, (1 << D)> W{};
    static constexpr int kDen = (D == 1 ? 8 : (D == 2 ? 64 : 512));
    static constexpr int kShift = 3 * D;

    TableBuilder()
    {
        const auto cfg = mrlbm::PredictionConfig::make(1);
        const int nst = kStencil<D>;
        for (int s = 0; s < (1 << D); ++s)
        {
            std::array<int, D> delta{};
            for (int i = 0; i < D; ++i)
                delta[i] = (s >> (D - 1 - i)) & 1;
            for (int o = 0; o < nst; ++o)
            {
                std::array<I64, 3> hot{};
                for (int a = 0; a < D; ++a)
                    hot[a] = stencil_off<D>(o, a);
                auto at = [&](std::array<I64, 3> off) { return (off == hot) ? 1.0 : 0.0; };
                const double w = mrlbm::predict<D>(at, delta, cfg);
                const double num = w * kDen;
                if (num != std::floor(num))
                    throw std::domain_error("table: non-dyadic prediction weight");
                W[s][o] = static_cast<I64>(num);
            }
        }
    }

    using Form = std::map<std::array<I64, D>, I128>; // level-l offset -> numerator

    // rec at depth dd above level l (dd = m - l), relative cell c (level m coords,
    // the leaf covers [0, 2^dd)^D).
    const Form& rec(int dd, const std::array<I64, D>& c, std::map<std::pair<int, std::array<I64, D>>, Form>& memo)
    {
        auto key = std::make_pair(dd, c);
        auto it = memo.find(key);
        if (it != memo.end())
            return it->second;
        Form out;
        if (dd == 0)
        {
            out[c] = 1; // numerator over 1
        }
        else
        {
            std::array<I64, D> p{};
            int s = 0;
            for (int i = 0; i < D; ++i)
            {
                p[i] = c[i] >> 1;
                s = (s << 1) | static_cast<int>(c[i] - 2 * p[i]);
            }
            const int nst = kStencil<D>;
            for (int o = 0; o < nst; ++o)
            {
                const I64 w = W[s][o];
                if (w == 0)
                    continue;
                std::array<I64, D> pc = p;
                for (int a = 0; a < D; ++a)
                    pc[a] += stencil_off<D>(o, a);
                const Form& sub = rec(dd - 1, pc, memo);
                for (const auto& [k, v] : sub)
                    out[k] += v * w; // numerators over kDen^dd
            }
        }
        return memo.emplace(key, std::move(out)).first->second;
    }

    // Exactness conditions of a table (Decision D.13): every level-l cell the
    // recursion touches must lie inside the domain (dep) and no cell it touches at
    // level l+1 may belong to the complete tree, i.e. their parents (par) must not
    // be internal.  Filled by build().
    std::vector<std::array<int, D>> last_dep, last_par;

    // side 0 = E = (B - eta) \ B, side 1 = A = B \ (B - eta)
    std::vector<std::pair<std::array<int, D>, double>> build(int g, const int32_t* eta, int side)
    {
        const I64 n = I64{1} << g;
        std::vector<std::array<I64, D>> cells;
        auto inB = [&](const std::array<I64, D>& x)
        {
            for (int i = 0; i < D; ++i)
                if (x[i] < 0 || x[i] >= n)
                    return false;
            return true;
        };
        // enumerate candidate finest cells in lexicographic order
        std::array<I64, D> lo{}, hi{};
        for (int i = 0; i < D; ++i)
        {
            lo[i] = -2;
            hi[i] = n + 2;
        }
        std::array<I64, D> x = lo;
        while (true)
        {
            std::array<I64, D> xe{};
            for (int i = 0; i < D; ++i)
                xe[i] = x[i] + eta[i];
            const bool member = side == 0 ? (inB(xe) && !inB(x)) : (inB(x) && !inB(xe));
            if (member)
                cells.push_back(x);
            int ax = D - 1;
            while (ax >= 0)
            {
                if (++x[ax] < hi[ax])
                    break;
                x[ax] = lo[ax];
                --ax;
            }
            if (ax < 0)
                break;
        }
        std::map<std::pair<int, std::array<I64, D>>, Form> memo;
        Form total;
        for (const auto& c : cells)
        {
            const Form& f = rec(g, c, memo);
            for (const auto& [k, v] : f)
                total[k] += v;
        }
        last_dep.clear();
        last_par.clear();
        std::map<std::array<I64, D>, int> par;
        for (const auto& [key, form] : memo)
        {
            if (key.first == 0)
            {
                std::array<int, D> o{};
                for (int i = 0; i < D; ++i)
                    o[i] = static_cast<int>(key.second[i]);
                last_dep.push_back(o);
            }
            else if (key.first == 1)
            {
                std::array<I64, D> pp{};
                for (int i = 0; i < D; ++i)
                    pp[i] = key.second[i] >> 1;
                par[pp] = 1;
            }
        }
        if (g == 0)
            for (const auto& c : cells)
            {
                std::array<int, D> o{};
                for (int i = 0; i < D; ++i)
                    o[i] = static_cast<int>(c[i]);
                last_dep.push_back(o);
            }
        for (const auto& [pp, one] : par)
        {
            std::array<int, D> o{};
            for (int i = 0; i < D; ++i)
                o[i] = static_cast<int>(pp[i]);
            last_par.push_back(o);
        }
        std::vector<std::pair<std::array<int, D>, double>> out;
        for (const auto& [k, v] : total)
        {
            if (v == 0)
                continue;
            // nearest double to the exact dyadic weight (Decision D.12)
            const double w = std::ldexp(static_cast<double>(v), -kShift * g);
            std::array<int, D> off{};
            for (int i = 0; i < D; ++i)
                off[i] = static_cast<int>(k[i]);
            out.emplace_back(off, w);
        }
        return out; // std::map order == lexicographic offsets
    }
};

// ---------------------------------------------------------------------------
// Equilibria (DESIGN.md Decisions D.18-D.21; PAPER.md:1143-1147,
// 1345-1348).  m is the full moment vector (conserved moments unchanged by
// collision); writes meq for every moment.
// ---------------------------------------------------------------------------
void equilibrium(const mrlbm_scheme_spec& sc, const double* m, double* meq)
{
    const double* P = sc.eq_params;
    switch (sc.equilibrium)
    {
        case MRLBM_EQ_BURGERS_D1Q2:
        {
            const double u = m[0];
            meq[0] = u;
            meq[1] = 0.5 * u * u;
            break;
        }
        case MRLBM_EQ_EULER_D1Q3X3:
        {
            const double gam = P[0];
            const double lam2 = sc.lambda * sc.lambda;
            const double rho = m[0], q = m[3], E = m[6];
            const double u = q / rho;
            const double p = (gam - 1.0) * (E - 0.5 * rho * u * u);
            const double F[3] = {q, q * u + p, u * (E + p)};
            const double U[3] = {rho, q, E};
            for (int i = 0; i < 3; ++i)
            {
                meq[3 * i + 0] = U[i];
                meq[3 * i + 1] = F[i];
                meq[3 * i + 2] = lam2 * U[i];
            }
            break;
        }
        case MRLBM_EQ_ADVECTION_D2Q4:
        {
            const double u = m[0];
            meq[0] = u;
            meq[1] = P[0] * u;
            meq[2] = P[1] * u;
            meq[3] = 0.0;
            break;
        }
        case MRLBM_EQ_EULER_D2Q4X4:
        {
            const double gam = P[0];
            const double rho = m[0], qx = m[4], qy = m[8], E = m[12];
            const double u = qx / rho;
            const double v = qy / rho;
            const double p = (gam - 1.0) * (E - 0.5 * rho * (u * u + v * v));
            const double Fx[4] = {qx, qx * u + p, qx * v, u * (E + p)};
            const double Fy[4] = {qy, qy * u, qy * v + p, v * (E + p)};
            const double U[4] = {rho, qx, qy, E};
            for (int i = 0; i < 4; ++i)
            {
                meq[4 * i + 0] = U[i];
                meq[4 * i + 1] = Fx[i];
                meq[4 * i + 2] = Fy[i];
                meq[4 * i + 3] = 0.0;
            }
            break;
        }
        case MRLBM_EQ_NS_D2Q9:
        {
            const double cs2 = P[0];
            const double rho = m[0], qx = m[1], qy = m[2];
            meq[0] = rho;
            meq[1] = qx;
            meq[2] = qy;
            if (P[1] == 0.0)
            {
                const double q2 = qx * qx + qy * qy;
                meq[3] = 3.0 * (-2.0 * cs2 * rho + q2 / rho);
                meq[6] = 9.0 * (cs2 * cs2 * rho - cs2 * q2 / rho);
            }
            else
            { // literal printed form: |q|/rho, c_s^4 without rho
                const double qn = std::sqrt(qx * qx + qy * qy);
                meq[3] = 3.0 * (-2.0 * cs2 * rho + qn / rho);
                meq[6] = 9.0 * (cs2 * cs2 - cs2 * qn / rho);
            }
            meq[4] = -3.0 * cs2 * qx;
            meq[5] = -3.0 * cs2 * qy;
            meq[7] = (qx * qx - qy * qy) / rho;
            meq[8] = qx * qy / rho;
            break;
        }
        case MRLBM_EQ_ADVECTION_D3Q6:
        {   // m^eq = (u, V_x u, V_y u, V_z u, 0, 0); eq_params = V
            const double u = m[0];
            meq[0] = u;
            meq[1] = P[0] * u;
            meq[2] = P[1] * u;
            meq[3] = P[2] * u;
            meq[4] = 0.0;
            meq[5] = 0.0;
            break;
        }
        default:
            throw std::invalid_argument("unknown equilibrium");
    }
}

template <int D>
class Oracle {
  public:
    using Idx = mrlbm::Index<D>;
    using Set = mrlbm::CellSet<D>;
    using CIdx = mrlbm::CellIndex<D>;

    struct Level {
        Set leaves, internal; // S(Lambda) and internal complete-tree nodes at this level
        CIdx li, ii;
        std::vector<double> lf, itf; // AoS values: [slot * q + h]
    };

    mrlbm_scheme_spec sc{};
    mrlbm_run_config rc{};
    int J0 = 0, J1 = 0, q = 0;
    mrlbm::DomainBox<D> box;
    bool per[D]{};
    mrlbm::PredictionConfig pcfg = mrlbm::PredictionConfig::make(1);
    mrlbm::DenseMatrix M, Minv;
    std::vector<Level> lev;                      // index m - J0
    std::vector<std::vector<std::pair<Idx, std::vector<double>>>> staged;
    bool committed = false;
    int opp[MRLBM_MAX_Q]{};
    // tables [gap][h][side] -> (offsets, weights), and their exactness sets
    std::vector<std::vector<std::array<std::vector<std::pair<std::array<int, D>, double>>, 2>>> tables;
    std::vector<std::vector<std::array<std::vector<std::array<int, D>>, 2>>> tdep, tpar;
    std::int64_t fallback_last = 0;
    std::int64_t leaf_updates = 0;
    std::string err;
    // obstacle force history: one (Fx, Fy) per step while tracking
    bool track_force = false;
    std::vector<double> force_hist;
    // near-threshold tie log (BASELINE north_star): steps since commit
    int step_no = 0;
    std::vector<mrlbm_tie_record> ties;

    // log a group metric within 1e-12 relative of a (positive) threshold; the
    // comparison metric >= threshold itself stays inclusive
    static bool tie_near(double metric, double thr)
    {
        return thr > 0.0 && std::fabs(metric - thr) <= 1e-12 * thr;
    }

    Oracle(const mrlbm_scheme_spec& s_, const mrlbm_run_config& r_) : sc(s_), rc(r_)
    {
        if (sc.d != D)
            throw std::invalid_argument("dimension mismatch");
        q = sc.q;
        if (q < 1 || q > MRLBM_MAX_Q)
            throw std::invalid_argument("q out of range");
        J0 = rc.j_min;
        J1 = rc.j_max;
        if (J0 < 0 || J1 <= J0 || J1 - J0 + 1 > MRLBM_MAX_LEVELS)
            throw std::invalid_argument("levels out of range");
        if (rc.gamma != 1 || rc.graduation != 1)
            throw std::invalid_argument("only gamma = graduation = 1 is supported");
        box.j_min = J0;
        for (int i = 0; i < D; ++i)
            box.base_cells[i] = rc.base_cells[i];
        for (int i = 0; i < D; ++i)
        {
            const bool a = rc.bc_kind[2 * i] == MRLBM_BC_PERIODIC;
            const bool b = rc.bc_kind[2 * i + 1] == MRLBM_BC_PERIODIC;
            if (a != b)
                throw std::invalid_argument("periodic must be set on both faces of an axis");
            per[i] = a;
        }
        M = mrlbm::DenseMatrix(q, q);
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < q; ++j)
                M(i, j) = sc.M[i * q + j];
        // M^-1 from the reference Gauss-Jordan (dense_matrix.hpp:58-113); the
        // descriptor's copy must agree bit for bit (the GPU uses the descriptor).
        Minv = M.inverse();
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < q; ++j)
                if (std::memcmp(&Minv(i, j), &sc.Minv[i * q + j], sizeof(double)) != 0)
                    throw std::invalid_argument("scheme Minv differs from DenseMatrix::inverse(M)");
        for (int h = 0; h < q; ++h)
        {
            opp[h] = -1;
            for (int k = 0; k < q; ++k)
            {
                bool ok = true;
                for (int i = 0; i < D; ++i)
                    ok = ok && sc.eta[k][i] == -sc.eta[h][i];
                // vectorial schemes: the opposite velocity inside the same block
                const int bs = q / sc.nblocks;
                ok = ok && (k / bs == h / bs);
                if (ok)
                {
                    opp[h] = k;
                    break;
                }
            }
        }
        lev.resize(J1 - J0 + 1);
        staged.resize(J1 - J0 + 1);
        TableBuilder<D> tb;
        tables.resize(J1 - J0 + 1);
        tdep.resize(J1 - J0 + 1);
        tpar.resize(J1 - J0 + 1);
        for (int g = 0; g <= J1 - J0; ++g)
        {
            tables[g].resize(q);
            tdep[g].resize(q);
            tpar[g].resize(q);
            for (int h = 0; h < q; ++h)
                for (int side = 0; side < 2; ++side)
                {
                    tables[g][h][side] = tb.build(g, sc.eta[h], side);
                    tdep[g][h][side] = tb.last_dep;
                    tpar[g][h][side] = tb.last_par;
                }
        }
    }

    // ---------------- geometry helpers ----------------
    Idx extent(int m) const { return box.extent(m); }

    // MR lookup rule outside the domain (Decision D.8): periodic wrap, else clamp.
    Idx wrapclamp(int m, Idx c) const
    {
        const Idx n = extent(m);
        for (int i = 0; i < D; ++i)
        {
            if (per[i])
            {
                c[i] %= n[i];
                if (c[i] < 0)
                    c[i] += n[i];
            }
            else if (c[i] < 0)
                c[i] = 0;
            else if (c[i] >= n[i])
                c[i] = n[i] - 1;
        }
        return c;
    }

    bool inside_or_periodic(int m, const Idx& c) const
    {
        const Idx n = extent(m);
        for (int i = 0; i < D; ++i)
            if (!per[i] && (c[i] < 0 || c[i] >= n[i]))
                return false;
        return true;
    }

    // set algebra image of a same-level set that may stick out of the domain:
    // clip non-periodic axes, wrap periodic ones (Decisions D.6, D.7)
    Set wrapclip(int m, const Set& s) const
    {
        const Idx n = extent(m);
        Set out;
        std::array<int, D> a{};
        for (int i = 0; i < D; ++i)
            a[i] = per[i] ? -1 : 0;
        while (true)
        {
            Idx shift{};
            for (int i = 0; i < D; ++i)
                shift[i] = static_cast<I64>(a[i]) * n[i];
            out.merge(s.translated(shift).clipped(box, m));
            int ax = D - 1;
            while (ax >= 0)
            {
                if (per[ax] && a[ax] < 1)
                {
                    ++a[ax];
                    break;
                }
                a[ax] = per[ax] ? -1 : 0;
                --ax;
            }
            if (ax < 0)
                break;
        }
        return out;
    }

    Set full_level(int m) const
    {
        Set s;
        const Idx n = extent(m);
        if constexpr (D == 1)
        {
            s.insert_run(Idx{0}, n[0]);
        }
        else if constexpr (D == 2)
        {
            for (I64 x = 0; x < n[0]; ++x)
                s.insert_run(Idx{x, 0}, n[1]);
        }
        else
        {
            for (I64 x = 0; x < n[0]; ++x)
                for (I64 y = 0; y < n[1]; ++y)
                    s.insert_run(Idx{x, y, 0}, n[2]);
        }
        return s;
    }

    // ---------------- value access on the current tree ----------------
    const double* value_R(int m, const Idx& c) const
    {
        const Level& L = lev[m - J0];
        if (auto s = L.li.slot(c))
            return &L.lf[*s * q];
        if (auto s = L.ii.slot(c))
            return &L.itf[*s * q];
        return nullptr;
    }

    // ---------------- loading ----------------
    void load(int level, I64 n, const int32_t* idx, const double* f)
    {
        if (level < J0 || level > J1)
            throw std::invalid_argument("load: level out of range");
        auto& st = staged[level - J0];
        st.clear();
        st.reserve(n);
        for (I64 i = 0; i < n; ++i)
        {
            Idx c{};
            for (int a = 0; a < D; ++a)
                c[a] = idx[i * D + a];
            std::vector<double> v(q);
            for (int h = 0; h < q; ++h)
                v[h] = f[h * n + i];
            st.emplace_back(c, std::move(v));
        }
    }

    void commit()
    {
        // refined sets from the loaded leaves (closure upwards), then derive and verify
        std::vector<Set> refined(J1 - J0);
        std::vector<Set> leafsets(J1 - J0 + 1);
        for (int m = J0; m <= J1; ++m)
            for (const auto& [c, v] : staged[m - J0])
            {
                if (!mrlbm::DomainBox<D>(box).contains(m, c))
                    throw std::invalid_argument("load: leaf outside the domain");
                leafsets[m - J0].insert(c);
            }
        for (int m = J1; m > J0; --m)
        {
            Set up = leafsets[m - J0].coarsened();
            if (m < J1)
                up.merge(refined[m - J0].coarsened());
            refined[m - 1 - J0].merge(up);
        }
        install_tree(refined);
        // verify partition and place values
        std::int64_t total = 0;
        for (int m = J0; m <= J1; ++m)
        {
            Level& L = lev[m - J0];
            const auto& st = staged[m - J0];
            if (static_cast<std::size_t>(L.leaves.cell_count()) != st.size())
                throw std::invalid_argument("load: leaves do not form a complete-leaf partition");
            L.lf.assign(st.size() * q, 0.0);
            for (const auto& [c, v] : st)
            {
                auto s = L.li.slot(c);
                if (!s)
                    throw std::invalid_argument("load: leaves do not form a complete-leaf partition");
                std::copy(v.begin(), v.end(), L.lf.begin() + *s * q);
            }
            total += st.size();
        }
        (void)total;
        for (auto& st : staged)
            st.clear();
        committed = true;
        step_no = 0;
        ties.clear();
    }

    // install a tree given refined sets per level (index m - J0, m < J1)
    void install_tree(const std::vector<Set>& refined)
    {
        for (int m = J0; m <= J1; ++m)
        {
            Level& L = lev[m - J0];
            Set R = (m == J0) ? full_level(m) : refined[m - 1 - J0].refined();
            if (m < J1)
            {
                L.internal = refined[m - J0];
                L.leaves = set_difference(R, L.internal);
            }
            else
            {
                L.internal = Set();
                L.leaves = R;
            }
            L.li = CIdx(L.leaves);
            L.ii = CIdx(L.internal);
            L.itf.assign(L.ii.size() * q, 0.0);
        }
    }

    std::vector<Set> current_refined() const
    {
        std::vector<Set> r(J1 - J0);
        for (int m = J0; m < J1; ++m)
            r[m - J0] = lev[m - J0].internal;
        return r;
    }

    // ---------------- the time step (Algorithm 1 body) ----
    void project_internal()
    {
        // bottom-up projection P_down (prediction.hpp:51-60)
        for (int m = J1 - 1; m >= J0; --m)
        {
            Level& L = lev[m - J0];
            std::vector<Idx> cells;
            L.internal.for_each_cell([&](const Idx& c) { cells.push_back(c); });
            OmpErr oe;
#pragma omp parallel for schedule(static)
            for (std::size_t i = 0; i < cells.size(); ++i)
                oe.run([&] {
                const Idx& p = cells[i];
                const auto ch = mrlbm::children(mrlbm::CellId<D>{m, p}, J1);
                const double* cv[1 << D];
                for (int s = 0; s < (1 << D); ++s)
                {
                    cv[s] = value_R(m + 1, ch[s].idx);
                    if (!cv[s])
                        throw std::logic_error("project: missing child");
                }
                const std::size_t slot = *L.ii.slot(p);
                for (int h = 0; h < q; ++h)
                {
                    std::array<double, (1 << D)> v{};
                    for (int s = 0; s < (1 << D); ++s)
                        v[s] = cv[s][h];
                    L.itf[slot * q + h] = mrlbm::project<D>(v);
                }
                });
            oe.rethrow();
        }
    }

    // gather the 3^D (or 5^D) same-level neighbourhood values with the MR rule
    template <int W, class Get>
    bool gather_box(int m, const Idx& center, std::vector<const double*>& out, Get&& get) const
    {
        constexpr int S = 2 * W + 1;
        constexpr int N = D == 1 ? S : (D == 2 ? S * S : S * S * S);
        out.resize(N);
        for (int o = 0; o < N; ++o)
        {
            Idx c = center;
            int r = o;
            for (int a = D - 1; a >= 0; --a)
            {
                c[a] += r % S - W;
                r /= S;
            }
            out[o] = get(m, wrapclamp(m, c));
            if (!out[o])
                return false;
        }
        return true;
    }

    double predict_from(const std::vector<const double*>& st3, const std::array<int, D>& delta, int h) const
    {
        // reference predict with an accessor over the prefetched 3^D stencil
        auto at = [&](std::array<I64, 3> off) -> double
        {
            int o = 0;
            for (int a = 0; a < D; ++a)
                o = o * 3 + static_cast<int>(off[a]) + 1;
            return st3[o][h];
        };
        return mrlbm::predict<D>(at, delta, pcfg);
    }

    void step()
    {
        if (!committed)
            throw std::logic_error("step before commit");
        const int nl = J1 - J0 + 1;
        // (1) projection of the old tree
        project_internal();

        // (2) details + group metric + T/H(b) flags
        std::vector<Set> keep(J1 - J0), Rn(J1 - J0);
        for (int m = J0; m < J1; ++m)
        {
            Level& L = lev[m - J0];
            const int l = m + 1; // level of the sibling group
            const double eps_l = std::ldexp(rc.epsilon, D * (l - J1));
            const double eps_b = std::ldexp(eps_l, rc.mu + D);
            std::vector<Idx> cells;
            L.internal.for_each_cell([&](const Idx& c) { cells.push_back(c); });
            std::vector<char> kflag(cells.size()), bflag(cells.size());
            OmpErr oe;
#pragma omp parallel
            {
                std::vector<const double*> st;
#pragma omp for schedule(static)
                for (std::size_t i = 0; i < cells.size(); ++i)
                    oe.run([&] {
                    const Idx& p = cells[i];
                    auto get = [&](int mm, const Idx& c) { return value_R(mm, c); };
                    if (!gather_box<1>(m, p, st, get))
                        throw std::logic_error("details: unresolved prediction stencil (grading)");
                    const auto ch = mrlbm::children(mrlbm::CellId<D>{m, p}, J1);
                    double metric = 0.0;
                    for (int s = 0; s < (1 << D); ++s)
                    {
                        std::array<int, D> delta{};
                        for (int a = 0; a < D; ++a)
                            delta[a] = (s >> (D - 1 - a)) & 1;
                        const double* cv = value_R(l, ch[s].idx);
                        for (int h = 0; h < q; ++h)
                        {
                            const double d = cv[h] - predict_from(st, delta, h);
                            const double ad = std::fabs(d);
                            if (ad > metric)
                                metric = ad;
                        }
                    }
                    kflag[i] = metric >= eps_l;
                    bflag[i] = (l > J0 && l < J1) && metric >= eps_b;
                    for (int which = 0; which < 2; ++which)
                    {
                        const double thr = which == 0 ? eps_l : eps_b;
                        if ((which == 0 || (l > J0 && l < J1)) && tie_near(metric, thr))
                        {
                            mrlbm_tie_record r{};
                            r.step = step_no + 1;
                            r.level = l;
                            for (int a = 0; a < D; ++a)
                                r.cell[a] = static_cast<int32_t>(p[a]);
                            r.which = which;
                            r.metric = metric;
                            r.threshold = thr;
#pragma omp critical(oracle_ties)
                            ties.push_back(r);
                        }
                    }
                    });
            }
            oe.rethrow();
            for (std::size_t i = 0; i < cells.size(); ++i)
            {
                if (kflag[i])
                    keep[m - J0].insert(cells[i]);
                if (bflag[i])
                {
                    // H(b): refine the 2^D children of every cell of the group
                    const auto ch = mrlbm::children(mrlbm::CellId<D>{m, cells[i]}, J1);
                    for (const auto& c : ch)
                        Rn[l - J0].insert(c.idx);
                }
            }
        }
        // T closure (Decision D.4): ancestors of kept groups are kept
        for (int m = J1 - 1; m > J0; --m)
            keep[m - 1 - J0].merge(keep[m - J0].coarsened());
        for (int m = J0; m < J1; ++m)
            Rn[m - J0].merge(keep[m - J0]);
        // H(a): (l, k - eta^h) for every cell of R(T)
        for (int l = J0 + 1; l <= J1; ++l)
        {
            const Set RT = keep[l - 1 - J0].refined();
            for (int h = 0; h < q; ++h)
            {
                Idx shift{};
                bool zero = true;
                for (int i = 0; i < D; ++i)
                {
                    shift[i] = -sc.eta[h][i];
                    zero = zero && shift[i] == 0;
                }
                if (zero)
                    continue;
                Rn[l - 1 - J0].merge(wrapclip(l, RT.translated(shift)).coarsened());
            }
        }
        // grading G: one fine->coarse sweep (Decision D.7)
        for (int m = J1 - 1; m > J0; --m)
            Rn[m - 1 - J0].merge(wrapclip(m, Rn[m - J0].dilated(1)).coarsened());

        // (3) transfer to the new tree (Decision D.24)
        std::vector<Level> old = std::move(lev);
        lev.assign(nl, Level{});
        install_tree(Rn);
        std::vector<Set> Rnew(nl);
        std::vector<CIdx> Ridx(nl);
        std::vector<std::vector<double>> Rval(nl);
        for (int m = J0; m <= J1; ++m)
        {
            Rnew[m - J0] = set_union(lev[m - J0].leaves, lev[m - J0].internal);
            Ridx[m - J0] = CIdx(Rnew[m - J0]);
            Rval[m - J0].assign(Ridx[m - J0].size() * q, 0.0);
            std::vector<Idx> cells;
            Rnew[m - J0].for_each_cell([&](const Idx& c) { cells.push_back(c); });
            const Level& O = old[m - J0];
            OmpErr oe;
#pragma omp parallel
            {
                std::vector<const double*> st;
#pragma omp for schedule(static)
                for (std::size_t i = 0; i < cells.size(); ++i)
                    oe.run([&] {
                    const Idx& c = cells[i];
                    double* dst = &Rval[m - J0][i * q];
                    const double* src = nullptr;
                    if (auto s = O.li.slot(c))
                        src = &O.lf[*s * q];
                    else if (auto s2 = O.ii.slot(c))
                        src = &O.itf[*s2 * q];
                    if (src)
                    {
                        std::copy(src, src + q, dst);
                        return;
                    }
                    if (m == J0)
                        throw std::logic_error("transfer: coarsest cell missing");
                    Idx p{};
                    std::array<int, D> delta{};
                    for (int a = 0; a < D; ++a)
                    {
                        p[a] = c[a] >> 1;
                        delta[a] = static_cast<int>(c[a] - 2 * p[a]);
                    }
                    auto get = [&](int mm, const Idx& cc) -> const double*
                    {
                        auto s = Ridx[mm - J0].slot(cc);
                        return s ? &Rval[mm - J0][*s * q] : nullptr;
                    };
                    if (!gather_box<1>(m - 1, p, st, get))
                        throw std::logic_error("transfer: unresolved stencil");
                    for (int h = 0; h < q; ++h)
                        dst[h] = predict_from(st, delta, h);
                    });
            }
            oe.rethrow();
            // split into leaves / internal (internal re-projected below)
            Level& L = lev[m - J0];
            L.lf.assign(L.li.size() * q, 0.0);
            L.leaves.for_each_cell(
                [&](const Idx& c)
                {
                    const std::size_t a = *L.li.slot(c), b = *Ridx[m - J0].slot(c);
                    std::copy(&Rval[m - J0][b * q], &Rval[m - J0][b * q] + q, &L.lf[a * q]);
                });
        }
        old.clear();
        // (4) internal values = projection of the new leaves (Decision D.25)
        project_internal();

        // (5) stream + collide on every new complete leaf
        stream_collide();
        leaf_updates += total_leaves();
    }

    std::int64_t total_leaves() const
    {
        std::int64_t n = 0;
        for (const auto& L : lev)
            n += L.li.size();
        return n;
    }

    using Memo = std::unordered_map<std::uint64_t, std::vector<double>>;

    std::uint64_t key(int m, const Idx& c) const
    {
        const Idx n = extent(m);
        std::uint64_t lin = 0;
        for (int i = 0; i < D; ++i)
            lin = lin * static_cast<std::uint64_t>(n[i]) + static_cast<std::uint64_t>(c[i]);
        return (static_cast<std::uint64_t>(m) << 56) | lin;
    }

    // zero-detail reconstruction f^^: R value if the cell is in
    // the complete tree, else prediction from the coarser level.  c is inside.
    const double* rec(int m, const Idx& c, Memo& memo) const
    {
        if (const double* v = value_R(m, c))
            return v;
        const std::uint64_t k = key(m, c);
        auto it = memo.find(k);
        if (it != memo.end())
            return it->second.data();
        if (m == J0)
            throw std::logic_error("rec: coarsest cell missing");
        Idx p{};
        std::array<int, D> delta{};
        for (int a = 0; a < D; ++a)
        {
            p[a] = c[a] >> 1;
            delta[a] = static_cast<int>(c[a] - 2 * p[a]);
        }
        std::vector<const double*> st(kStencil<D>);
        for (int o = 0; o < kStencil<D>; ++o)
        {
            Idx cc = p;
            for (int a = 0; a < D; ++a)
                cc[a] += stencil_off<D>(o, a);
            st[o] = rec(m - 1, wrapclamp(m - 1, cc), memo);
        }
        std::vector<double> v(q);
        for (int h = 0; h < q; ++h)
            v[h] = predict_from(st, delta, h);
        return memo.emplace(k, std::move(v)).first->second.data();
    }

    // value of the complete leaf covering finest cell c (direct evaluation)
    const double* covering_leaf(const Idx& cfine) const
    {
        for (int m = J1; m >= J0; --m)
        {
            Idx a{};
            for (int i = 0; i < D; ++i)
                a[i] = cfine[i] >> (J1 - m);
            const Level& L = lev[m - J0];
            if (auto s = L.li.slot(a))
                return &L.lf[*s * q];
        }
        throw std::logic_error("covering leaf not found");
    }

    // finest-level E / A cells of leaf (l, k) for velocity eta, lexicographic
    void rim_cells(int l, const Idx& k, const int32_t* eta, int side, std::vector<Idx>& out) const
    {
        out.clear();
        const int g = J1 - l;
        const I64 n = I64{1} << g;
        Idx lo{}, hi{};
        for (int i = 0; i < D; ++i)
        {
            lo[i] = k[i] * n - 1;
            hi[i] = (k[i] + 1) * n + 1;
        }
        auto inB = [&](const Idx& x)
        {
            for (int i = 0; i < D; ++i)
                if (x[i] < k[i] * n || x[i] >= (k[i] + 1) * n)
                    return false;
            return true;
        };
        Idx x = lo;
        while (true)
        {
            Idx xe{};
            for (int i = 0; i < D; ++i)
                xe[i] = x[i] + eta[i];
            const bool member = side == 0 ? (inB(xe) && !inB(x)) : (inB(x) && !inB(xe));
            if (member)
                out.push_back(x);
            int ax = D - 1;
            while (ax >= 0)
            {
                if (++x[ax] < hi[ax])
                    break;
                x[ax] = lo[ax];
                --ax;
            }
            if (ax < 0)
                break;
        }
    }

    void stream_collide()
    {
        const Idx nfine = extent(J1);
        std::int64_t nfb = 0;
        const bool trk = track_force && rc.obstacle == 1;
        double force[2] = {0.0, 0.0};
        for (int l = J0; l <= J1; ++l)
        {
            Level& L = lev[l - J0];
            const int g = J1 - l;
            const double scale = std::ldexp(1.0, D * (l - J1));
            std::vector<Idx> cells;
            L.leaves.for_each_cell([&](const Idx& c) { cells.push_back(c); });
            std::vector<double> out(cells.size() * q);
            std::vector<double> fc(trk ? cells.size() * 2 : 0, 0.0);
            std::vector<char> fb(cells.size(), 0);
            OmpErr oe;
#pragma omp parallel reduction(+ : nfb)
            {
                Memo memo;
                std::vector<Idx> rim;
                std::vector<double> f(q), mm(q), meq(q), mp(q), fs(q);
#pragma omp for schedule(dynamic, 256)
                for (std::size_t i = 0; i < cells.size(); ++i)
                    oe.run([&] {
                    const Idx& k = cells[i];
                    const double* fstar = &L.lf[*L.li.slot(k) * q];
                    bool any_fb = false;
                    for (int h = 0; h < q; ++h)
                    {
                        double sums[2] = {0.0, 0.0};
                        for (int side = 0; side < 2; ++side)
                        {
                            // table exactness (Decision D.13): dependency cells inside
                            // (or periodic), parents of the level-(l+1) funnel not internal
                            bool dom_ok = true, par_ok = true;
                            for (const auto& o : tdep[g][h][side])
                            {
                                Idx c = k;
                                for (int a = 0; a < D; ++a)
                                    c[a] += o[a];
                                if (!inside_or_periodic(l, c))
                                {
                                    dom_ok = false;
                                    break;
                                }
                            }
                            for (const auto& o : tpar[g][h][side])
                            {
                                if (!dom_ok)
                                    break;
                                Idx c = k;
                                for (int a = 0; a < D; ++a)
                                    c[a] += o[a];
                                if (L.ii.slot(wrapclamp(l, c)))
                                    par_ok = false;
                            }
                            double s = 0.0;
                            if (dom_ok && (par_ok || g == 1))
                            {
                                for (const auto& [off, w] : tables[g][h][side])
                                {
                                    Idx c = k;
                                    for (int a = 0; a < D; ++a)
                                        c[a] += off[a];
                                    s += w * rec(l, wrapclamp(l, c), memo)[h];
                                }
                                if (!par_ok)
                                {
                                    // gap 1 with finer neighbours (Decision D.13b, "add
                                    // the proper detail information"): the table sums the predicted
                                    // rim values; add the detail of every rim cell that is a leaf
                                    any_fb = true;
                                    rim_cells(l, k, sc.eta[h], side, rim);
                                    for (const auto& x : rim)
                                    {
                                        const Idx xc = wrapclamp(J1, x);
                                        const double* v = value_R(J1, xc);
                                        if (!v)
                                            continue;
                                        Idx p{};
                                        std::array<int, D> delta{};
                                        for (int a = 0; a < D; ++a)
                                        {
                                            p[a] = xc[a] >> 1;
                                            delta[a] = static_cast<int>(xc[a] - 2 * p[a]);
                                        }
                                        std::vector<const double*> st(kStencil<D>);
                                        for (int o = 0; o < kStencil<D>; ++o)
                                        {
                                            Idx cc = p;
                                            for (int a = 0; a < D; ++a)
                                                cc[a] += stencil_off<D>(o, a);
                                            st[o] = rec(l, wrapclamp(l, cc), memo);
                                        }
                                        s += v[h] - predict_from(st, delta, h);
                                    }
                                }
                            }
                            else
                            {
                                any_fb = true;
                                rim_cells(l, k, sc.eta[h], side, rim);
                                for (const auto& x : rim)
                                    s += side == 0 ? rim_value(x, h, fstar, nfine, memo) : rec(J1, x, memo)[h];
                            }
                            sums[side] = s;
                        }
                        f[h] = fstar[h] + scale * (sums[0] - sums[1]);
                    }
                    fb[i] = any_fb;
                    nfb += any_fb ? 1 : 0;
                    // collide (Decision D.24)
                    M.multiply(f.data(), mm.data());
                    equilibrium(sc, mm.data(), meq.data());
                    for (int h = 0; h < q; ++h)
                        mp[h] = (1.0 - sc.s[h]) * mm[h] + sc.s[h] * meq[h];
                    Minv.multiply(mp.data(), fs.data());
                    if (rc.obstacle == 1)
                    {
                        const double alpha = obstacle_blend(l, k, fs.data());
                        if (trk && alpha > 0.0)
                            force_terms(l, alpha, mp.data(), &fc[2 * i]);
                    }
                    for (int h = 0; h < q; ++h)
                    {
                        if (!std::isfinite(fs[h]))
                            throw std::domain_error("non-finite population after collision");
                        out[i * q + h] = fs[h];
                    }
                    });
            }
            oe.rethrow();
            // write after all leaves of this level have read their stencils: but
            // stencils also read other levels -> defer the swap until all levels done
            pending.push_back(std::move(out));
            // obstacle force: level by level, leaves in CellIndex order
            for (std::size_t i = 0; i < fc.size() / 2; ++i)
            {
                force[0] = force[0] + fc[2 * i];
                force[1] = force[1] + fc[2 * i + 1];
            }
        }
        for (int l = J0; l <= J1; ++l)
            lev[l - J0].lf = std::move(pending[l - J0]);
        pending.clear();
        fallback_last = nfb;
        ++step_no;
        if (trk)
        {
            force_hist.push_back(force[0]);
            force_hist.push_back(force[1]);
        }
    }

    // Force on the obstacle (SPEC.md:468-476 design decision "force via momentum
    // exchange of the obstacle blend"): the momentum the blend removes from a leaf per
    // unit time, alpha * q * |cell| / dt with q = the post-collision momentum moments
    // (conserved by the collision) and dt = dx_J / lambda (acoustic scaling).
    void force_terms(int l, double alpha, const double* mp, double* out) const
    {
        const double area = std::ldexp(1.0, -D * l);
        const double dt = std::ldexp(1.0, -J1) / sc.lambda;
        for (int a = 0; a < 2; ++a)
            out[a] = ((alpha * mp[1 + a]) * area) / dt;
    }
    std::vector<std::vector<double>> pending;

    // E-rim value: reconstruction inside the domain, boundary rule outside
    double rim_value(const Idx& x, int h, const double* fstar_leaf, const Idx& nfine, Memo& memo) const
    {
        int face = -1;
        for (int i = 0; i < D && face < 0; ++i)
        {
            if (per[i])
                continue;
            if (x[i] < 0)
                face = 2 * i;
            else if (x[i] >= nfine[i])
                face = 2 * i + 1;
        }
        if (face < 0)
            return rec(J1, wrapclamp(J1, x), memo)[h];
        const int kind = rc.bc_kind[face];
        switch (kind)
        {
            case MRLBM_BC_COPY:
                return covering_leaf(wrapclamp(J1, x))[h];
            case MRLBM_BC_BOUNCE_BACK:
                return fstar_leaf[opp_checked(h)];
            case MRLBM_BC_ANTI_BOUNCE_BACK:
                return -fstar_leaf[opp_checked(h)];
            case MRLBM_BC_VELOCITY_BOUNCE_BACK:
                return fstar_leaf[opp_checked(h)] + rc.bc_add[face][h];
            default:
                throw std::invalid_argument("bad boundary kind");
        }
    }

    int opp_checked(int h) const
    {
        if (opp[h] < 0)
            throw std::invalid_argument("bounce-back needs an opposite velocity");
        return opp[h];
    }

    // config 5 obstacle: alpha by
    // sub-sampling, f <- alpha feq0 + (1 - alpha) f
    double obstacle_blend(int l, const Idx& k, double* fs) const
    {
        const int ns = rc.obstacle_subsamples;
        const double dx = std::ldexp(1.0, -l);
        const double r2 = rc.obstacle_radius * rc.obstacle_radius;
        double x0[D], x1[D];
        for (int i = 0; i < D; ++i)
        {
            x0[i] = rc.origin[i] + static_cast<double>(k[i]) * dx;
            x1[i] = x0[i] + dx;
        }
        // bounding-box rejection (exact in dyadics)
        for (int i = 0; i < D; ++i)
            if (x1[i] < rc.obstacle_center[i] - rc.obstacle_radius || x0[i] > rc.obstacle_center[i] + rc.obstacle_radius)
                return 0.0;
        int cnt = 0;
        for (int a = 0; a < ns; ++a)
            for (int b = 0; b < (D == 1 ? 1 : ns); ++b)
            {
                const double sx = rc.origin[0] + (static_cast<double>(k[0]) + (a + 0.5) / ns) * dx;
                double rr = (sx - rc.obstacle_center[0]) * (sx - rc.obstacle_center[0]);
                if (D >= 2)
                {
                    const double sy = rc.origin[1] + (static_cast<double>(k[D - 1]) + (b + 0.5) / ns) * dx;
                    rr = rr + (sy - rc.obstacle_center[1]) * (sy - rc.obstacle_center[1]);
                }
                cnt += rr < r2;
            }
        if (cnt == 0)
            return 0.0;
        const double alpha = static_cast<double>(cnt) / (D == 1 ? ns : ns * ns);
        for (int h = 0; h < q; ++h)
            fs[h] = alpha * rc.obstacle_feq[h] + (1.0 - alpha) * fs[h];
        return alpha;
    }

    std::int64_t level_count(int m) const { return lev[m - J0].li.size(); }

    void read(int m, int32_t* idx, double* f) const
    {
        const Level& L = lev[m - J0];
        const std::size_t n = L.li.size();
        std::size_t i = 0;
        L.leaves.for_each_cell(
            [&](const Idx& c)
            {
                if (idx)
                    for (int a = 0; a < D; ++a)
                        idx[i * D + a] = static_cast<int32_t>(c[a]);
                if (f)
                    for (int h = 0; h < q; ++h)
                        f[h * n + i] = L.lf[i * q + h];
                ++i;
            });
    }

    std::int64_t internal_count(int m) const { return lev[m - J0].ii.size(); }

    // f^^ of the current state on the full finest grid: internal
    // values re-projected from the current leaves (the next step's project_internal
    // computes the same), then rec() per finest cell; out = SoA q x n, lexicographic.
    void reconstruct_finest(double* out)
    {
        project_internal();
        Memo memo;
        const Idx n = extent(J1);
        std::int64_t total = 1;
        for (int i = 0; i < D; ++i)
            total *= n[i];
        for (std::int64_t lin = 0; lin < total; ++lin)
        {
            Idx c{};
            std::int64_t r = lin;
            for (int i = D - 1; i >= 0; --i)
            {
                c[i] = r % n[i];
                r /= n[i];
            }
            const double* v = rec(J1, c, memo);
            for (int h = 0; h < q; ++h)
                out[h * total + lin] = v[h];
        }
    }
};

struct Handle {
    int d = 0;
    std::unique_ptr<Oracle<1>> o1;
    std::unique_ptr<Oracle<2>> o2;
    std::unique_ptr<Oracle<3>> o3;
    std::string err;
};

template <class Fn>
int guard(Handle* h, Fn&& fn)
{
    try
    {
        fn();
        return MRLBM_OK;
    }
    catch (const std::invalid_argument& e)
    {
        h->err = e.what();
        return MRLBM_ERR_CONFIG;
    }
    catch (const std::domain_error& e)
    {
        h->err = e.what();
        return MRLBM_ERR_NUMERIC;
    }
    catch (const std::exception& e)
    {
        h->err = e.what();
        return MRLBM_ERR_CAPACITY;
    }
}

} // namespace

extern "C" {

int oracle_create(const mrlbm_scheme_spec* sc, const mrlbm_run_config* rc, void** out)
{
    auto* h = new Handle();
    h->d = sc->d;
    const int st = guard(h,
                         [&]
                         {
                             if (sc->d == 1)
                                 h->o1 = std::make_unique<Oracle<1>>(*sc, *rc);
                             else if (sc->d == 2)
                                 h->o2 = std::make_unique<Oracle<2>>(*sc, *rc);
                             else if (sc->d == 3)
                                 h->o3 = std::make_unique<Oracle<3>>(*sc, *rc);
                             else
                                 throw std::invalid_argument("d must be 1, 2 or 3");
                         });
    if (st != MRLBM_OK)
    {
        static thread_local std::string last;
        last = h->err;
        delete h;
        *out = nullptr;
        return st;
    }
    *out = h;
    return MRLBM_OK;
}

#define ORACLE_DISPATCH(h, call)                                                                   \
    guard(h, [&] {                                                                                 \
        if (h->o1)                                                                                 \
            h->o1->call;                                                                           \
        else if (h->o2)                                                                            \
            h->o2->call;                                                                           \
        else                                                                                       \
            h->o3->call;                                                                           \
    })

int oracle_load_leaves(void* p, int level, int64_t n, const int32_t* idx, const double* f)
{
    auto* h = static_cast<Handle*>(p);
    return ORACLE_DISPATCH(h, load(level, n, idx, f));
}

int oracle_commit(void* p)
{
    auto* h = static_cast<Handle*>(p);
    return ORACLE_DISPATCH(h, commit());
}

int oracle_step(void* p, int nsteps)
{
    auto* h = static_cast<Handle*>(p);
    for (int i = 0; i < nsteps; ++i)
    {
        const int st = ORACLE_DISPATCH(h, step());
        if (st != MRLBM_OK)
            return st;
    }
    return MRLBM_OK;
}

int oracle_level_count(void* p, int level, int64_t* n)
{
    auto* h = static_cast<Handle*>(p);
    return guard(h, [&] { *n = h->o1 ? h->o1->level_count(level) : h->o2 ? h->o2->level_count(level) : h->o3->level_count(level); });
}

int oracle_internal_count(void* p, int level, int64_t* n)
{
    auto* h = static_cast<Handle*>(p);
    return guard(h, [&] { *n = h->o1 ? h->o1->internal_count(level) : h->o2 ? h->o2->internal_count(level) : h->o3->internal_count(level); });
}

int oracle_read_leaves(void* p, int level, int32_t* idx, double* f)
{
    auto* h = static_cast<Handle*>(p);
    return ORACLE_DISPATCH(h, read(level, idx, f));
}

int oracle_reconstruct_finest(void* p, double* f)
{
    auto* h = static_cast<Handle*>(p);
    return ORACLE_DISPATCH(h, reconstruct_finest(f));
}

int64_t oracle_fallback_leaves(void* p)
{
    auto* h = static_cast<Handle*>(p);
    return h->o1 ? h->o1->fallback_last : h->o2 ? h->o2->fallback_last : h->o3->fallback_last;
}

int oracle_set_force_tracking(void* p, int on)
{
    auto* h = static_cast<Handle*>(p);
    return guard(h, [&] {
        if (!h->o2)
            throw std::invalid_argument("force tracking needs the 2D obstacle configuration");
        if (h->o2->rc.obstacle != 1)
            throw std::invalid_argument("force tracking needs an obstacle (run config obstacle = 1)");
        h->o2->track_force = on != 0;
        h->o2->force_hist.clear();
    });
}

// per-step obstacle forces recorded since tracking was enabled: n = number of steps
int oracle_force_history(void* p, double* fx, double* fy, int cap, int* n)
{
    auto* h = static_cast<Handle*>(p);
    return guard(h, [&] {
        const std::vector<double>& v = h->o2 ? h->o2->force_hist : std::vector<double>{};
        const int k = static_cast<int>(v.size() / 2);
        for (int i = 0; i < k && i < cap; ++i)
        {
            fx[i] = v[2 * i];
            fy[i] = v[2 * i + 1];
        }
        *n = k;
    });
}

// tie log since commit (or the last reset), sorted by (step, level, cell, which)
int oracle_tie_log(void* p, mrlbm_tie_record* out, int cap, int64_t* n, int reset)
{
    auto* h = static_cast<Handle*>(p);
    return guard(h, [&] {
        std::vector<mrlbm_tie_record>& t = h->o1 ? h->o1->ties : h->o2 ? h->o2->ties : h->o3->ties;
        std::sort(t.begin(), t.end(), [](const mrlbm_tie_record& a, const mrlbm_tie_record& b) {
            if (a.step != b.step) return a.step < b.step;
            if (a.level != b.level) return a.level < b.level;
            for (int k = 0; k < 3; ++k)
                if (a.cell[k] != b.cell[k]) return a.cell[k] < b.cell[k];
            return a.which < b.which;
        });
        *n = static_cast<int64_t>(t.size());
        for (int i = 0; out && i < cap && i < static_cast<int>(t.size()); ++i)
            out[i] = t[i];
        if (reset)
            t.clear();
    });
}

const char* oracle_last_error(void* p)
{
    return static_cast<Handle*>(p)->err.c_str();
}

void oracle_destroy(void* p)
{
    delete static_cast<Handle*>(p);
}

int oracle_set_threads(int n)
{
    omp_set_num_threads(n);
    return omp_get_max_threads();
}

// table export (pull formulation) for cross-checking the product's tables
int oracle_stream_table(int d, int gap, const int32_t eta[3], int side, int cap, int32_t* offsets, double* weights, int* n)
{
    try
    {
        if (d == 1)
        {
            TableBuilder<1> tb;
            auto t = tb.build(gap, eta, side);
            if (static_cast<int>(t.size()) > cap)
                return MRLBM_ERR_CAPACITY;
            for (std::size_t i = 0; i < t.size(); ++i)
            {
                offsets[i] = t[i].first[0];
                weights[i] = t[i].second;
            }
            *n = static_cast<int>(t.size());
        }
        else if (d == 2)
        {
            TableBuilder<2> tb;
            auto t = tb.build(gap, eta, side);
            if (static_cast<int>(t.size()) > cap)
                return MRLBM_ERR_CAPACITY;
            for (std::size_t i = 0; i < t.size(); ++i)
            {
                offsets[2 * i] = t[i].first[0];
                offsets[2 * i + 1] = t[i].first[1];
                weights[i] = t[i].second;
            }
            *n = static_cast<int>(t.size());
        }
        else
        {
            TableBuilder<3> tb;
            auto t = tb.build(gap, eta, side);
            if (static_cast<int>(t.size()) > cap)
                return MRLBM_ERR_CAPACITY;
            for (std::size_t i = 0; i < t.size(); ++i)
            {
                for (int a = 0; a < 3; ++a)
                    offsets[3 * i + a] = t[i].first[a];
                weights[i] = t[i].second;
            }
            *n = static_cast<int>(t.size());
        }
        return MRLBM_OK;
    }
    catch (...)
    {
        return MRLBM_ERR_NUMERIC;
    }
}

int oracle_stream_table_sets(int d, int gap, const int32_t eta[3], int side, int cap, int32_t* dep, int* ndep,
                             int32_t* par, int* npar)
{
    try
    {
        auto emit = [&](const auto& tb)
        {
            if (static_cast<int>(tb.last_dep.size()) > cap || static_cast<int>(tb.last_par.size()) > cap)
                return MRLBM_ERR_CAPACITY;
            for (std::size_t i = 0; i < tb.last_dep.size(); ++i)
                for (int a = 0; a < d; ++a)
                    dep[i * d + a] = tb.last_dep[i][a];
            for (std::size_t i = 0; i < tb.last_par.size(); ++i)
                for (int a = 0; a < d; ++a)
                    par[i * d + a] = tb.last_par[i][a];
            *ndep = static_cast<int>(tb.last_dep.size());
            *npar = static_cast<int>(tb.last_par.size());
            return MRLBM_OK;
        };
        if (d == 1)
        {
            TableBuilder<1> tb;
            tb.build(gap, eta, side);
            return emit(tb);
        }
        if (d == 3)
        {
            TableBuilder<3> tb;
            tb.build(gap, eta, side);
            return emit(tb);
        }
        TableBuilder<2> tb;
        tb.build(gap, eta, side);
        return emit(tb);
    }
    catch (...)
    {
        return MRLBM_ERR_NUMERIC;
    }
}


} // extern "C"

// ---------------------------------------------------------------------------
// Independent scheme / run descriptors and initial data for the five BASELINE
// configurations, written from BASELINE.json configs[0..4] and the decisions
// ledger (D.2, D.9, D.14-D.22), NOT from the product's builder
// (paper_2103_02903_b200/csrc/host_configs.cpp).  tests/test_descriptors.py pins
// every field of the product's descriptors against these, and bench.py's
// reference arm builds its run from these alone (no product library loaded).
// M^-1 = the reference DenseMatrix::inverse (dense_matrix.hpp:58-113); equilibrium
// populations = the reference DenseMatrix::multiply (dense_matrix.hpp:42-54) of
// M^-1 and this file's equilibrium() (used by the oracle's collision as well).
// ---------------------------------------------------------------------------
namespace {

struct Blk {
    int first, size; // population range of one block of a (block-diagonal) vectorial scheme
};

// D2Q4 change of basis: rows 1, lambda xi_x, lambda xi_y, lambda^2 (xi_x^2 - xi_y^2)
// over the velocities (1,0), (0,1), (-1,0), (0,-1)
void d2q4_rows(double lam, double r[4][4])
{
    static const int ex[4] = {1, 0, -1, 0}, ey[4] = {0, 1, 0, -1};
    for (int j = 0; j < 4; ++j)
    {
        r[0][j] = 1.0;
        r[1][j] = lam * ex[j];
        r[2][j] = lam * ey[j];
        r[3][j] = lam * lam * (ex[j] * ex[j] - ey[j] * ey[j]);
    }
}

int build_descriptors(int id, int jmax_override, double eps_override, mrlbm_scheme_spec* sc, mrlbm_run_config* rc)
{
    *sc = mrlbm_scheme_spec{};
    *rc = mrlbm_run_config{};
    rc->gamma = 1;            // prediction stencil gamma = 1 (BASELINE, all configs)
    rc->graduation = 1;       // grading box half-width = gamma (D.9)
    rc->obstacle_subsamples = 16;
    rc->j_min = 2;
    auto set_eta = [&](int h, int x, int y) { sc->eta[h][0] = x; sc->eta[h][1] = y; };
    // entries are stored as v + 0.0: structural zeros are +0.0 (no -0.0 from x * 0)
    auto Mset = [&](int i, int j, double v) { sc->M[i * sc->q + j] = v + 0.0; };
    double rho0 = 1.0, u0 = 0.0, radius = 0.0, Re = 0.0;
    if (id == 1)
    {   // D1Q2 Burgers, [-3,3], levels 2..10, lambda 1, s 1.5, eps 1e-4, outflow (D.2, D.18)
        sc->d = 1; sc->q = 2; sc->nblocks = 1; sc->equilibrium = MRLBM_EQ_BURGERS_D1Q2; sc->lambda = 1.0;
        set_eta(0, 1, 0); set_eta(1, -1, 0);
        Mset(0, 0, 1.0); Mset(0, 1, 1.0); Mset(1, 0, sc->lambda); Mset(1, 1, -sc->lambda);
        sc->s[1] = 1.5;
        rc->j_max = 10; rc->base_cells[0] = 24; rc->origin[0] = -3.0; rc->epsilon = 1e-4; rc->mu = 0;
        rc->bc_kind[0] = rc->bc_kind[1] = MRLBM_BC_COPY;
    }
    else if (id == 2)
    {   // three coupled D1Q3 (rho, q, E), lambda 3, s 1.9, eps 1e-4, levels 2..14 (D.19)
        sc->d = 1; sc->q = 9; sc->nblocks = 3; sc->equilibrium = MRLBM_EQ_EULER_D1Q3X3; sc->lambda = 3.0;
        sc->eq_params[0] = 1.4;
        const double lam = sc->lambda;
        for (Blk b : {Blk{0, 3}, Blk{3, 3}, Blk{6, 3}})
        {
            const int v[3] = {0, 1, -1};
            for (int j = 0; j < 3; ++j)
            {
                set_eta(b.first + j, v[j], 0);
                Mset(b.first + 0, b.first + j, 1.0);
                Mset(b.first + 1, b.first + j, lam * v[j]);
                Mset(b.first + 2, b.first + j, v[j] == 0 ? 0.0 : lam * lam);
            }
            sc->s[b.first + 1] = sc->s[b.first + 2] = 1.9;
        }
        rc->j_max = 14; rc->base_cells[0] = 4; rc->epsilon = 1e-4; rc->mu = 0;
        rc->bc_kind[0] = rc->bc_kind[1] = MRLBM_BC_COPY;
    }
    else if (id == 3 || id == 4)
    {   // D2Q4 advection (a, b) = (1, 1), periodic (D.20) / D2Q4^4 Euler, lambda 4, outflow (D.21)
        const int nb = id == 3 ? 1 : 4;
        sc->d = 2; sc->q = 4 * nb; sc->nblocks = nb;
        sc->equilibrium = id == 3 ? MRLBM_EQ_ADVECTION_D2Q4 : MRLBM_EQ_EULER_D2Q4X4;
        sc->lambda = id == 3 ? 1.0 : 4.0;
        if (id == 3) { sc->eq_params[0] = 1.0; sc->eq_params[1] = 1.0; }
        else sc->eq_params[0] = 1.4;
        double r[4][4];
        d2q4_rows(sc->lambda, r);
        static const int ex[4] = {1, 0, -1, 0}, ey[4] = {0, 1, 0, -1};
        for (int b = 0; b < nb; ++b)
            for (int i = 0; i < 4; ++i)
            {
                set_eta(4 * b + i, ex[i], ey[i]);
                for (int j = 0; j < 4; ++j)
                    Mset(4 * b + i, 4 * b + j, r[i][j]);
                sc->s[4 * b + i] = i == 0 ? 0.0 : 1.9;
            }
        rc->j_max = id == 3 ? 9 : 11;
        rc->base_cells[0] = rc->base_cells[1] = 4;
        rc->epsilon = id == 3 ? 1e-4 : 1e-3;
        rc->mu = 0;
        for (int f = 0; f < 4; ++f)
            rc->bc_kind[f] = id == 3 ? MRLBM_BC_PERIODIC : MRLBM_BC_COPY;
    }
    else if (id == 5)
    {   // D2Q9 Lallemand-Luo past a cylinder (D.14-D.17)
        sc->d = 2; sc->q = 9; sc->nblocks = 1; sc->equilibrium = MRLBM_EQ_NS_D2Q9; sc->lambda = 1.0;
        const double lam = sc->lambda;
        // xi^h: 0; lambda (cos, sin)(pi/2 (h-1)); lambda (cos, sin)(pi/2 (h-5) + pi/4) / |.| -> unit lattice
        const int vx[9] = {0, 1, 0, -1, 0, 1, -1, -1, 1}, vy[9] = {0, 0, 1, 0, -1, 1, 1, -1, -1};
        for (int h = 0; h < 9; ++h)
        {
            set_eta(h, vx[h], vy[h]);
            const double x = vx[h], y = vy[h], n2 = x * x + y * y;
            // rows of PAPER.md:1334-1343 as polynomials of the velocity, lambda powers applied
            const double row[9] = {1.0,
                                   lam * x,
                                   lam * y,
                                   lam * lam * (3.0 * n2 - 4.0),
                                   lam * lam * lam * (3.0 * n2 - 5.0) * x,
                                   lam * lam * lam * (3.0 * n2 - 5.0) * y,
                                   lam * lam * lam * lam * (9.0 * n2 * n2 / 2.0 - 21.0 * n2 / 2.0 + 4.0),
                                   lam * lam * (x * x - y * y),
                                   lam * lam * x * y};
            for (int i = 0; i < 9; ++i)
                Mset(i, h, row[i]);
        }
        const double cs2 = lam * lam / 3.0; // c_s = lambda / sqrt(3)
        sc->eq_params[0] = cs2;
        sc->eq_params[1] = 0.0;             // |q|^2 / rho form (D.17)
        rho0 = 1.0; u0 = 0.05; Re = 1200.0; radius = 0.0625;
        rc->j_max = 12; rc->base_cells[0] = 8; rc->base_cells[1] = 4; rc->epsilon = 1e-4; rc->mu = 1;
        rc->bc_kind[0] = rc->bc_kind[2] = rc->bc_kind[3] = MRLBM_BC_VELOCITY_BOUNCE_BACK; // inlet, bottom, top
        rc->bc_kind[1] = MRLBM_BC_COPY;                                                // outlet
        rc->obstacle = 1;
        rc->obstacle_center[0] = 0.3125;
        rc->obstacle_center[1] = 0.5;
        rc->obstacle_radius = radius;
    }
    else if (id == 6)
    {   // D3Q6 advection of a sphere indicator (D.28):
        // J 1..8, mu = 2, eps = 1e-3, lambda = 1, S = diag(0, s1, s1, s1, s2, s2), s1 = 1.4, s2 = 1,
        // unit cube [-3/8, 5/8]^3 (2 cells per axis at level 1), V = (1/4, 1/4, 1/4) (inside the positivity
        // bound |V_a| <= lambda / 3 of the D3Q6 equilibrium; V = 1/2 blows up), copy boundaries
        sc->d = 3; sc->q = 6; sc->nblocks = 1; sc->equilibrium = MRLBM_EQ_ADVECTION_D3Q6; sc->lambda = 1.0;
        const double lam = sc->lambda;
        for (int h = 0; h < 6; ++h)
        {   // xi^h = lambda cos(pi h) e_{h / 2}: +x, -x, +y, -y, +z, -z
            const int ax = h / 2, sg = (h % 2 == 0) ? 1 : -1;
            sc->eta[h][ax] = sg;
            Mset(0, h, 1.0);
            Mset(1 + ax, h, lam * sg);
        }
        // rows 4, 5: lambda^2 (1,1,-1,-1,0,0), lambda^2 (1,1,0,0,-1,-1)
        const double r4[6] = {1, 1, -1, -1, 0, 0}, r5[6] = {1, 1, 0, 0, -1, -1};
        for (int h = 0; h < 6; ++h)
        {
            Mset(4, h, lam * lam * r4[h]);
            Mset(5, h, lam * lam * r5[h]);
        }
        sc->s[1] = sc->s[2] = sc->s[3] = 1.4;
        sc->s[4] = sc->s[5] = 1.0;
        sc->eq_params[0] = sc->eq_params[1] = sc->eq_params[2] = 0.25;
        rc->j_min = 1; rc->j_max = 8; rc->epsilon = 1e-3; rc->mu = 2;
        for (int a = 0; a < 3; ++a)
        {
            rc->base_cells[a] = 2;
            rc->origin[a] = -0.375;
        }
        for (int f = 0; f < 6; ++f)
            rc->bc_kind[f] = MRLBM_BC_COPY;
    }
    else
        return MRLBM_ERR_CONFIG;
    if (jmax_override > 0)
    {
        if (jmax_override <= rc->j_min)
            return MRLBM_ERR_CONFIG;
        rc->j_max = jmax_override;
    }
    if (eps_override >= 0.0)
        rc->epsilon = eps_override;
    const int q = sc->q;
    if (id == 5)
    {
        // s1 pinned (D.17); s2 from the viscosity:
        // s2 = (1/2 + mu_visc / (c_s^2 dt rho0))^-1, mu_visc = rho0 u0 L / Re, L = 2 r, dt = dx_J / lambda
        const double cs2 = sc->eq_params[0];
        const double L = 2.0 * radius;
        const double mu_visc = rho0 * u0 * L / Re;
        const double dt = std::ldexp(1.0, -rc->j_max) / sc->lambda;
        const double s2 = 1.0 / (0.5 + mu_visc / (cs2 * dt * rho0));
        for (int h = 3; h < 7; ++h)
            sc->s[h] = 1.5;
        sc->s[7] = sc->s[8] = s2;
        // moving-wall (Ladd) term 2 w_h rho0 (xi_h . u_w) / c_s^2 with u_w = (u0, 0) on the
        // velocity bounce-back faces (D.14); D2Q9 weights 4/9, 1/9, 1/36
        for (int f = 0; f < 4; ++f)
            for (int h = 0; h < 9; ++h)
            {
                const int n1 = std::abs(sc->eta[h][0]) + std::abs(sc->eta[h][1]);
                const double w = n1 == 0 ? 4.0 / 9 : (n1 == 1 ? 1.0 / 9 : 1.0 / 36);
                const double xu = sc->lambda * sc->eta[h][0] * u0;
                rc->bc_add[f][h] = rc->bc_kind[f] == MRLBM_BC_VELOCITY_BOUNCE_BACK ? 2.0 * w * rho0 * xu / cs2 : 0.0;
            }
    }
    mrlbm::DenseMatrix M(q, q);
    for (int i = 0; i < q; ++i)
        for (int j = 0; j < q; ++j)
            M(i, j) = sc->M[i * q + j];
    const mrlbm::DenseMatrix Mi = M.inverse();
    for (int i = 0; i < q; ++i)
        for (int j = 0; j < q; ++j)
            sc->Minv[i * q + j] = Mi(i, j);
    if (id == 5)
    {   // obstacle target M^-1 m^eq(rho0, 0, 0)
        double m[MRLBM_MAX_Q] = {rho0, 0.0, 0.0}, meq[MRLBM_MAX_Q] = {};
        equilibrium(*sc, m, meq);
        Mi.multiply(meq, rc->obstacle_feq);
    }
    return MRLBM_OK;
}

// splitmix64 finaliser -> uniform double in [-1, 1) (D.16: 53 high bits)
double unit_sm64(std::uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

} // namespace

extern "C" {

int oracle_build_config(int id, int jmax_override, double eps_override, mrlbm_scheme_spec* sc, mrlbm_run_config* rc)
{
    try
    {
        return build_descriptors(id, jmax_override, eps_override, sc, rc);
    }
    catch (...)
    {
        return MRLBM_ERR_CONFIG;
    }
}

// f = M^-1 m^eq(conserved moments of the datum at the finest cell centre) (D.22),
// SoA q x N, cells in CellIndex order (axis 0 slow)
int oracle_initial_finest(int id, const mrlbm_scheme_spec* sc, const mrlbm_run_config* rc, uint64_t seed, double* f)
{
    const int q = sc->q, d = sc->d, J = rc->j_max;
    const std::int64_t nx = rc->base_cells[0] << (J - rc->j_min);
    const std::int64_t ny = d >= 2 ? (rc->base_cells[1] << (J - rc->j_min)) : 1;
    const std::int64_t nz = d == 3 ? (rc->base_cells[2] << (J - rc->j_min)) : 1;
    const std::int64_t N = nx * ny * nz;
    const double h = std::ldexp(1.0, -J);
    mrlbm::DenseMatrix Mi(q, q);
    for (int i = 0; i < q; ++i)
        for (int j = 0; j < q; ++j)
            Mi(i, j) = sc->Minv[i * q + j];
    const int bs = q / sc->nblocks;
    auto energy = [](double rho, double u, double v, double p, double gam) {
        return p / (gam - 1.0) + 0.5 * rho * (u * u + v * v);
    };
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < N; ++i)
    {
        const std::int64_t ix = i / (ny * nz), iy = (i / nz) % ny, iz = i % nz;
        const double x = rc->origin[0] + (static_cast<double>(ix) + 0.5) * h;
        const double y = rc->origin[1] + (static_cast<double>(iy) + 0.5) * h;
        const double z = rc->origin[2] + (static_cast<double>(iz) + 0.5) * h;
        double U[4] = {0, 0, 0, 0}; // conserved variables, one per block
        switch (id)
        {
            case 1: U[0] = std::max(0.0, 1.0 - std::fabs(x)); break;
            case 2:
            {   // Lax shock tube, (rho, u, p)_L = (0.445, 0.698, 3.528), _R = (0.5, 0, 0.571), jump at 0.5
                const double rho = x < 0.5 ? 0.445 : 0.5, u = x < 0.5 ? 0.698 : 0.0, p = x < 0.5 ? 3.528 : 0.571;
                U[0] = rho; U[1] = rho * u; U[2] = energy(rho, u, 0.0, p, sc->eq_params[0]);
                break;
            }
            case 3: U[0] = ((x - 0.5) * (x - 0.5) + (y - 0.5) * (y - 0.5) <= 0.04) ? 1.0 : 0.0; break;
            case 4:
            {   // quadrant states (rho, u, v, p): NE, NW, SW, SE
                static const double st[4][4] = {{1.5, 0.0, 0.0, 1.5}, {0.5323, 1.206, 0.0, 0.3},
                                                {0.138, 1.206, 1.206, 0.029}, {0.5323, 0.0, 1.206, 0.3}};
                const int k = (x > 0.5 && y > 0.5) ? 0 : (x < 0.5 && y > 0.5) ? 1 : (x < 0.5 && y < 0.5) ? 2 : 3;
                U[0] = st[k][0]; U[1] = st[k][0] * st[k][1]; U[2] = st[k][0] * st[k][2];
                U[3] = energy(st[k][0], st[k][1], st[k][2], st[k][3], sc->eq_params[0]);
                break;
            }
            case 5: U[0] = 1.0; U[1] = 0.0; U[2] = 1.0 * (1e-3 * unit_sm64(seed ^ static_cast<std::uint64_t>(i))); break;
            case 6: U[0] = (x * x + y * y + z * z <= 0.15 * 0.15) ? 1.0 : 0.0; break;
            default: break;
        }
        double m[MRLBM_MAX_Q] = {}, meq[MRLBM_MAX_Q] = {}, fl[MRLBM_MAX_Q] = {};
        if (id == 5)
        {
            m[0] = U[0]; m[1] = U[1]; m[2] = U[2];
        }
        else
            for (int b = 0; b < sc->nblocks; ++b)
                m[b * bs] = U[b];
        equilibrium(*sc, m, meq);
        Mi.multiply(meq, fl);
        for (int k = 0; k < q; ++k)
            f[k * N + i] = fl[k];
    }
    return (id >= 1 && id <= 6) ? MRLBM_OK : MRLBM_ERR_CONFIG;
}

} // extern "C"
