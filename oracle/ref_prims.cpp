// ref_prims.cpp — C-ABI shim exposing the REFERENCE's own primitives
// (/root/reference/proj/core/include/mrlbm/*.hpp, included, never copied) so the
// tests can pin the oracle and the product against upstream code.
// TEST INFRASTRUCTURE ONLY; built into oracle/_ref/ by oracle/Makefile.
#include <mrlbm/cell.hpp>
#include <mrlbm/cell_set.hpp>
#include <mrlbm/dense_matrix.hpp>
#include <mrlbm/prediction.hpp>
#include <mrlbm/rational.hpp>

#include <cstdint>
#include <cstring>

extern "C" {

// predict<D> (prediction.hpp:143-173) on a dense (2g+1)^D stencil, row-major,
// last axis fastest; delta = child selector.
double ref_predict(int d, int gamma, const double* stencil, const int* delta)
{
    const auto cfg = mrlbm::PredictionConfig::make(gamma);
    const int w = 2 * gamma + 1;
    auto at = [&](std::array<std::int64_t, 3> o) -> double
    {
        std::int64_t lin = 0;
        for (int i = 0; i < d; ++i)
            lin = lin * w + (o[i] + gamma);
        return stencil[lin];
    };
    if (d == 1)
        return mrlbm::predict<1>(at, std::array<int, 1>{delta[0]}, cfg);
    if (d == 2)
        return mrlbm::predict<2>(at, std::array<int, 2>{delta[0], delta[1]}, cfg);
    return mrlbm::predict<3>(at, std::array<int, 3>{delta[0], delta[1], delta[2]}, cfg);
}

// project<D> (prediction.hpp:51-60)
double ref_project(int d, const double* v)
{
    if (d == 1)
        return mrlbm::project<1>({v[0], v[1]});
    if (d == 2)
        return mrlbm::project<2>({v[0], v[1], v[2], v[3]});
    std::array<double, 8> a{};
    std::memcpy(a.data(), v, sizeof(a));
    return mrlbm::project<3>(a);
}

// derive_prediction_weights (prediction.hpp:199-309) -> num/den pairs
int ref_derive_weights(int gamma, std::int64_t* num, std::int64_t* den)
{
    try
    {
        auto c = mrlbm::derive_prediction_weights(gamma);
        for (std::size_t i = 0; i < c.size(); ++i)
        {
            num[i] = c[i].num();
            den[i] = c[i].den();
        }
        return static_cast<int>(c.size());
    }
    catch (...)
    {
        return -1;
    }
}

// PredictionConfig::make(gamma).c (prediction.hpp:22-45)
int ref_prediction_coeffs(int gamma, double* c)
{
    const auto cfg = mrlbm::PredictionConfig::make(gamma);
    for (int a = 0; a < 3; ++a)
        c[a] = cfg.c[a];
    return gamma;
}

// DenseMatrix::inverse (dense_matrix.hpp:58-113), row-major n x n
int ref_inverse(int n, const double* a, double* out)
{
    try
    {
        mrlbm::DenseMatrix m(n, n);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                m(i, j) = a[i * n + j];
        auto inv = m.inverse();
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                out[i * n + j] = inv(i, j);
        return 0;
    }
    catch (...)
    {
        return -1;
    }
}

// DenseMatrix::multiply (dense_matrix.hpp:42-54)
void ref_multiply(int n, const double* a, const double* x, double* y)
{
    mrlbm::DenseMatrix m(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            m(i, j) = a[i * n + j];
    m.multiply(x, y);
}

// children / parent (cell.hpp:80-116), 2D
int ref_children2(int level, std::int64_t kx, std::int64_t ky, int jmax, std::int64_t* out)
{
    try
    {
        auto ch = mrlbm::children(mrlbm::CellId<2>{level, {kx, ky}}, jmax);
        for (int s = 0; s < 4; ++s)
        {
            out[2 * s] = ch[s].idx[0];
            out[2 * s + 1] = ch[s].idx[1];
        }
        return 0;
    }
    catch (...)
    {
        return -1;
    }
}

int ref_parent2(int level, std::int64_t kx, std::int64_t ky, int jmin, std::int64_t* out)
{
    try
    {
        auto p = mrlbm::parent(mrlbm::CellId<2>{level, {kx, ky}}, jmin);
        out[0] = p.idx[0];
        out[1] = p.idx[1];
        return p.level;
    }
    catch (...)
    {
        return -1;
    }
}

// CellIndex slot order (cell_set.hpp:333-354): insert cells, return slots
int ref_cellindex_slots2(int n, const std::int64_t* xy, std::int64_t* slots)
{
    mrlbm::CellSet<2> s;
    for (int i = 0; i < n; ++i)
        s.insert({xy[2 * i], xy[2 * i + 1]});
    mrlbm::CellIndex<2> idx(s);
    for (int i = 0; i < n; ++i)
    {
        auto sl = idx.slot({xy[2 * i], xy[2 * i + 1]});
        slots[i] = sl ? static_cast<std::int64_t>(*sl) : -1;
    }
    return static_cast<int>(idx.size());
}

} // extern "C"
