// interp.cu -- per-cell Lagrange spread (interpolation.hpp:84-92) fused with
// the forward z-contraction of the collapsed SKP operator, and the backward
// z-expansion fused with the gather (interpolation.hpp:95-105) and the
// zero-mode correction (parallel.hpp:284-287).
//
// One CTA owns a column of cells (c0, c1, z-segment). Particles were sorted
// by flattened cell index, so a column's particles are one contiguous range
// and each cell's grid accumulates in shared memory / registers: no global
// atomics, and every sum runs in a fixed order (bit-identical re-runs).
#include "internal.h"
#include "trace.h"

namespace kb {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxL = 16;   // CLI range --order 2..16 (tools/kpme.cpp:343)
constexpr int kChunk = 64;  // particles staged per spread step

// CellGrid::axis_lo / axis_hi (geometry.hpp:90-98)
__device__ __forceinline__ double cell_lo(const Geometry& g, int a, int i) {
    return g.center[a] - g.radius + 2.0 * g.radius * i / g.K[a];
}
__device__ __forceinline__ double cell_hi(const Geometry& g, int a, int i) {
    return g.center[a] - g.radius + 2.0 * g.radius * (i + 1) / g.K[a];
}

// Same exact key arithmetic as the sort (internal.h, geometry.hpp:141-148).
__device__ __forceinline__ int axis_cell(double p, double c, double r, int K, double y) {
    return exact_axis_cell(p, c, r, K, __dmul_rn(2.0, r), y);
}

// Equispaced Lagrange weights on [lo, hi] (lagrange_weights_1d,
// interpolation.hpp:20-36) in prefix/suffix-product form:
// w_k = c_k * prod_{j<k}(t - t_j) * prod_{j>k}(t - t_j), c_k = 1/prod(t_k - t_j).
__device__ __forceinline__ void lagrange(const Geometry& g, const double* lc, double lo,
                                         double hi, double y, double* w,
                                         unsigned long long* bad) {
    const int L = g.L;
    const double slack = 1e-12 * (hi - lo);  // tensor_weights, interpolation.hpp:47-49
    if (y < lo - slack || y > hi + slack) atomicOr(&bad[1], 1ull);
    const double t = (y - 0.5 * (hi + lo)) / (0.5 * (hi - lo));
    const double step = 2.0 / (L - 1);
    double pre = 1.0;
#pragma unroll
    for (int k = 0; k < kMaxL; ++k)
        if (k < L) {
            w[k] = pre;
            pre *= t - (-1.0 + step * k);
        }
    double suf = 1.0;
#pragma unroll
    for (int k = kMaxL - 1; k >= 0; --k)
        if (k < L) {
            w[k] *= suf * lc[k];
            suf *= t - (-1.0 + step * k);
        }
}

struct ColumnRange {
    int col, seg, c0, c1, zb, ze;
};
__device__ __forceinline__ ColumnRange column_range(const Geometry& g, int S) {
    ColumnRange r;
    const int lc = blockIdx.x / S, ny = g.y_hi - g.y_lo;  // column of the plan's cell block
    r.seg = blockIdx.x % S;
    r.c0 = g.x_lo + lc / ny;
    r.c1 = g.y_lo + lc % ny;
    r.col = r.c0 * g.K[1] + r.c1;
    const int span = g.z_hi - g.z_lo;
    r.zb = g.z_lo + (int)((long long)r.seg * span / S);
    r.ze = g.z_lo + (int)((long long)(r.seg + 1) * span / S);
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_spread_fwd(ColumnArgs a, int want_fwd) {
    const Geometry& g = a.g;
    const int L = g.L, L2 = L * L, L3 = L2 * L, R = g.R, tid = threadIdx.x;
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    double* phi = sm;                 // L^3       current cell grid
    double* t1 = phi + L3;            // L^2 x R   column partial of W2 phi
    double* w2s = t1 + L2 * R;        // R x L     W2 slice of the current cell
    double* wb = w2s + R * L;         // kChunk x 3L particle weights (axis 0 * q)
    __shared__ double lc[kMaxL];
    __shared__ double red[kThreads];
    if (tid < L) {
        // c_k = 1 / prod_{j != k} (t_k - t_j), t_j = -1 + 2j/(L-1)
        double d = 1.0;
        for (int j = 0; j < L; ++j)
            if (j != tid) d *= (2.0 * tid / (L - 1)) - (2.0 * j / (L - 1));
        lc[tid] = 1.0 / d;
    }
    for (int e = tid; e < L2 * R; e += kThreads) t1[e] = 0.0;
    const double lo0 = cell_lo(g, 0, cr.c0), hi0 = cell_hi(g, 0, cr.c0);
    const double lo1 = cell_lo(g, 1, cr.c1), hi1 = cell_hi(g, 1, cr.c1);
    double qsum = 0.0;
    __syncthreads();

    for (int c2 = cr.zb; c2 < cr.ze; ++c2) {
        const int cell = (cr.c0 * g.K[1] + cr.c1) * g.K[2] + c2;
        if (MODE == SPREAD_PARTICLES) {
            const int s0 = a.start[cell], s1 = a.start[cell + 1];
            if (s1 == s0) {  // empty cell: phi = 0, contributes nothing
                if (a.phi_cells)
                    for (int node = tid; node < L3; node += kThreads)
                        a.phi_cells[(int64_t)cell * L3 + node] = 0.0;
                continue;
            }
            const double lo2 = cell_lo(g, 2, c2), hi2 = cell_hi(g, 2, c2);
            double acc[kMaxL];  // ceil(L^3 / kThreads) <= 16 nodes per thread
#pragma unroll
            for (int k = 0; k < kMaxL; ++k) acc[k] = 0.0;
            for (int base = s0; base < s1; base += kChunk) {
                const int cnt = min(kChunk, s1 - base);
                __syncthreads();
                for (int j = tid; j < cnt; j += kThreads) {
                    const double4 p = a.sp[base + j];
                    double w[kMaxL];
                    double* dst = wb + j * 3 * L;
                    lagrange(g, lc, lo0, hi0, p.x, w, a.bad);
                    for (int k = 0; k < L; ++k) dst[k] = p.w * w[k];
                    lagrange(g, lc, lo1, hi1, p.y, w, a.bad);
                    for (int k = 0; k < L; ++k) dst[L + k] = w[k];
                    lagrange(g, lc, lo2, hi2, p.z, w, a.bad);
                    for (int k = 0; k < L; ++k) dst[2 * L + k] = w[k];
                    qsum += p.w;
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < kMaxL; ++k) {
                    const int node = tid + k * kThreads;
                    if (node < L3) {
                        const int i = node / L2, jj = (node / L) % L, kk = node % L;
                        double s = acc[k];
                        for (int j = 0; j < cnt; ++j) {
                            const double* w = wb + j * 3 * L;
                            s = fma(w[i] * w[L + jj], w[2 * L + kk], s);
                        }
                        acc[k] = s;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kMaxL; ++k) {
                const int node = tid + k * kThreads;
                if (node < L3) {
                    phi[node] = acc[k];
                    if (a.phi_cells) a.phi_cells[(int64_t)cell * L3 + node] = acc[k];
                }
            }
        } else {
            for (int node = tid; node < L3; node += kThreads)
                phi[node] = a.phi_cells[(int64_t)cell * L3 + node];
        }
        if (!want_fwd) continue;
        for (int e = tid; e < R * L; e += kThreads)
            w2s[e] = a.W2[(int64_t)(e / L) * g.n[2] + c2 * L + e % L];
        __syncthreads();
        // t1[(i,j), r] += sum_l W2[r, c2*L + l] * phi[i, j, l]
        for (int e = tid; e < L2 * R; e += kThreads) {
            const int ij = e / R, r = e % R;
            double s = 0.0;
            for (int l = 0; l < L; ++l) s = fma(w2s[r * L + l], phi[ij * L + l], s);
            t1[e] += s;
        }
        __syncthreads();
    }
    if (want_fwd) {
        double* dst = a.T1 + (int64_t)cr.seg * g.n[0] * g.n[1] * R;
        for (int e = tid; e < L2 * R; e += kThreads) {
            const int ij = e / R, r = e % R, i = ij / L, j = ij % L;
            dst[((int64_t)(cr.c0 * L + i) * g.n[1] + cr.c1 * L + j) * R + r] = t1[e];
        }
    }
    if (MODE == SPREAD_PARTICLES && a.colq) {
        red[tid] = qsum;
        __syncthreads();
        for (int o = kThreads / 2; o > 0; o >>= 1) {
            if (tid < o) red[tid] += red[tid + o];
            __syncthreads();
        }
        if (tid == 0) a.colq[(int64_t)cr.seg * g.K[0] * g.K[1] + cr.col] = red[0];
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_bwd_gather(ColumnArgs a, int cells_per_batch) {
    const Geometry& g = a.g;
    const int L = g.L, L2 = L * L, L3 = L2 * L, R = g.R, tid = threadIdx.x;
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    double* b2s = sm;             // L^2 x R   column block of B2
    double* psi = b2s + L2 * R;   // cells_per_batch x L^3
    __shared__ double lc[kMaxL];
    if (tid < L) {
        double d = 1.0;
        for (int j = 0; j < L; ++j)
            if (j != tid) d *= (2.0 * tid / (L - 1)) - (2.0 * j / (L - 1));
        lc[tid] = 1.0 / d;
    }
    if (MODE != GATHER_FROM_CELLS)
        for (int e = tid; e < L2 * R; e += kThreads) {
            const int ij = e / R, r = e % R, i = ij / L, j = ij % L;
            b2s[e] = a.B2[((int64_t)(cr.c0 * L + i) * g.n[1] + cr.c1 * L + j) * R + r];
        }
    const double lo0 = cell_lo(g, 0, cr.c0), hi0 = cell_hi(g, 0, cr.c0);
    const double lo1 = cell_lo(g, 1, cr.c1), hi1 = cell_hi(g, 1, cr.c1);
    const double corr = a.corr ? *a.corr : 0.0;
    __syncthreads();

    for (int cb0 = cr.zb; cb0 < cr.ze; cb0 += cells_per_batch) {
        const int cb1 = min(cr.ze, cb0 + cells_per_batch);
        const int cell0 = (cr.c0 * g.K[1] + cr.c1) * g.K[2] + cb0;
        for (int e = tid; e < (cb1 - cb0) * L3; e += kThreads) {
            const int b = e / L3, node = e % L3, c2 = cb0 + b;
            if (MODE == GATHER_FROM_CELLS) {
                psi[e] = a.psi_cells[(int64_t)(cell0 + b) * L3 + node];
            } else {
                const int ij = node / L, k = node % L;
                double s = 0.0;
                for (int r = 0; r < R; ++r)
                    s = fma(a.W2[(int64_t)r * g.n[2] + c2 * L + k], b2s[ij * R + r], s);
                psi[e] = s;
                if (a.psi_cells) a.psi_cells[(int64_t)(cell0 + b) * L3 + node] = s;
            }
        }
        __syncthreads();
        if (MODE != PSI_ONLY) {
            const int s0 = a.start[cell0], s1 = a.start[cell0 + (cb1 - cb0)];
            for (int s = s0 + tid; s < s1; s += kThreads) {
                const double4 p = a.sp[s];
                const int c2 = axis_cell(p.z, g.center[2], g.radius, g.K[2], g.inv_diam);
                const double* ps = psi + (c2 - cb0) * L3;
                double w0[kMaxL], w1[kMaxL], w2[kMaxL];
                lagrange(g, lc, lo0, hi0, p.x, w0, a.bad);
                lagrange(g, lc, lo1, hi1, p.y, w1, a.bad);
                lagrange(g, lc, cell_lo(g, 2, c2), cell_hi(g, 2, c2), p.z, w2, a.bad);
                double z = 0.0;
                for (int i = 0; i < L; ++i) {
                    double zi = 0.0;
                    for (int j = 0; j < L; ++j) {
                        const double* row = ps + (i * L + j) * L;
                        double zij = 0.0;
#pragma unroll
                        for (int k = 0; k < kMaxL; ++k)
                            if (k < L) zij = fma(w2[k], row[k], zij);
                        zi = fma(w1[j], zij, zi);
                    }
                    z = fma(w0[i], zi, z);
                }
                a.out[a.perm[s]] = z - corr;
            }
        }
        __syncthreads();
    }
}


// ---------------------------------------------------------------------------
// Compile-time-L kernels (the hot path). Register arrays stay in registers.
// ---------------------------------------------------------------------------

template <int L>
__device__ __forceinline__ void lagrange_t(const double* lc, double lo, double hi, double y,
                                           double (&w)[L], unsigned long long* bad) {
    const double slack = 1e-12 * (hi - lo);  // tensor_weights, interpolation.hpp:47-49
    if (y < lo - slack || y > hi + slack) atomicOr(&bad[1], 1ull);
    const double t = (y - 0.5 * (hi + lo)) / (0.5 * (hi - lo));
    constexpr double step = 2.0 / (L - 1);
    double pre = 1.0;
#pragma unroll
    for (int k = 0; k < L; ++k) {
        w[k] = pre;
        pre *= t - (-1.0 + step * k);
    }
    double suf = 1.0;
#pragma unroll
    for (int k = L - 1; k >= 0; --k) {
        w[k] *= suf * lc[k];
        suf *= t - (-1.0 + step * k);
    }
}

__device__ __forceinline__ void lagrange_consts(int L, double* lc) {
    const int k = threadIdx.x;
    if (k < L) {
        double d = 1.0;
        for (int j = 0; j < L; ++j)
            if (j != k) d *= (2.0 * k / (L - 1)) - (2.0 * j / (L - 1));
        lc[k] = 1.0 / d;
    }
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// c_k = 1 / prod_{j != k} (t_k - t_j) for equispaced t_j = -1 + 2j/(L-1),
// evaluated at compile time.
template <int L>
struct LagrangeConsts {
    double c[L];
    constexpr LagrangeConsts() : c() {
        for (int k = 0; k < L; ++k) {
            double d = 1.0;
            for (int j = 0; j < L; ++j)
                if (j != k) d *= (2.0 * k / (L - 1)) - (2.0 * j / (L - 1));
            c[k] = 1.0 / d;
        }
    }
};

// Division-free Lagrange weights: t = (y - mid) * inv_half with mid, inv_half
// precomputed once per cell axis (same nodes as lagrange_weights_1d,
// interpolation.hpp:20-36; rounding differs by a few ulps).
template <int L>
__device__ __forceinline__ void lagrange_fast(const double* /*lc*/, double lo, double hi,
                                              double mid, double inv_half, double y,
                                              double (&w)[L], unsigned long long* bad) {
    constexpr LagrangeConsts<L> C;
    const double slack = 1e-12 * (hi - lo);  // tensor_weights, interpolation.hpp:47-49
    if (y < lo - slack || y > hi + slack) atomicOr(&bad[1], 1ull);
    const double t = (y - mid) * inv_half;
    constexpr double step = 2.0 / (L - 1);
    double d[L];
#pragma unroll
    for (int k = 0; k < L; ++k) d[k] = t - (-1.0 + step * k);
    double pre = C.c[0];
#pragma unroll
    for (int k = 0; k < L; ++k) {
        w[k] = pre;
        if (k + 1 < L) pre = pre * d[k] * (C.c[k + 1 < L ? k + 1 : 0] / C.c[k]);
    }
    double suf = 1.0;
#pragma unroll
    for (int k = L - 1; k >= 0; --k) {
        w[k] *= suf;
        suf *= d[k];
    }
}

// First cell c in [cb, ce] with start[c] >= target (start is non-decreasing),
// found by the whole warp 32 cells at a time.
__device__ __forceinline__ int warp_lower_bound(const int32_t* start, int cb, int ce, int target,
                                                int lane) {
    for (int base = cb; base <= ce; base += 32) {
        const int c = base + lane;
        const bool hit = c <= ce && start[c] >= target;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (m) return base + __ffs(m) - 1;
    }
    return ce;
}

// Powers t^a of the cell-local coordinate t = (y - mid) / half (monomial hot
// path), with the same out-of-cell check as tensor_weights.
template <int L>
__device__ __forceinline__ void powers(double lo, double hi, double mid, double inv_half,
                                       double y, double (&w)[L], unsigned long long* bad) {
    const double slack = 1e-12 * (hi - lo);
    if (y < lo - slack || y > hi + slack) atomicOr(&bad[1], 1ull);
    const double t = (y - mid) * inv_half;
    w[0] = 1.0;
#pragma unroll
    for (int k = 1; k < L; ++k) w[k] = w[k - 1] * t;
}

struct CellAxis {
    double lo, hi, mid, inv;
};
__device__ __forceinline__ CellAxis cell_axis_tab(const double4* tab, int i) {
    const double4 v = tab[i];
    return CellAxis{v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ CellAxis cell_axis(const Geometry& g, int a, int i) {
    CellAxis c;
    c.lo = cell_lo(g, a, i);
    c.hi = cell_hi(g, a, i);
    c.mid = 0.5 * (c.hi + c.lo);
    c.inv = 1.0 / (0.5 * (c.hi - c.lo));
    return c;
}

// Spread on FP64 tensor cores. For one cell,
//     phi[i][(j,k)] = sum_p (q_p w0_p[i]) (w1_p[j] w2_p[k])
// is an (L x L^2) = (L x P)(P x L^2) GEMM over the cell's particles. Each
// warp owns whole cells; per 16-particle chunk a lane pair (l, l+16) builds
// one particle's A row (q w0, 8 padded) and B row (w1 (x) w2, NT*8 padded)
// particle-contiguous in shared memory, then 4 k-steps of m8n8k4 DMMA
// accumulate phi in registers. The finished grid is contracted with the
// cell's W2 slice, T1c[(i,j)][r] = sum_k phi[(i,j)][k] W2[r][c2 L + k], on
// DMMA as well, into the warp's column partial of T1.
#ifndef SPREAD_MINB
#define SPREAD_MINB 3
#endif
#ifndef SPREAD_CH
#define SPREAD_CH 16
#endif
#ifndef SPREAD_SKIP
#define SPREAD_SKIP 0  // profiling ablations only: 1 DMMA loop, 2 staging, 4 prep, 8 contraction
#endif

template <int L>
struct SpreadTile {
    static constexpr int L2 = L * L;
    static constexpr int NT = (L2 + 7) / 8;   // n-tiles over (j,k)
    static constexpr int MT2 = (L2 + 7) / 8;  // m-tiles of the contraction (rows (i,j))
    static constexpr int KS2 = (L + 3) / 4;   // k-steps of the contraction
    static constexpr int LDK = KS2 * 4;       // phi[(i,j)][k] row stride
    static constexpr int CH = SPREAD_CH;      // particles staged per chunk (16: lane pairs)
    static constexpr int LDP = CH + 4;        // staged row stride (conflict-free fragments)
    static constexpr int NW = 4;              // warps per CTA
    static constexpr int stage = (8 + NT * 8) * LDP;
    static_assert(MT2 * 8 * LDK <= stage, "phi must fit in the staging area");
};

__host__ __device__ constexpr int spread_epilogue_doubles(int L, int R) {
    return L * L * R + L * R * R + 2 * R * L;
}

template <int L>
__host__ __device__ constexpr int spread_warp_doubles(int R) {
    return SpreadTile<L>::stage + SpreadTile<L>::MT2 * 8 * ((R + 7) / 8) * 8;
}


// Staging rows that are identically zero (A rows >= L, B rows >= L^2); the
// chunk loop never writes them, so they are cleared once per cell reuse.
template <int L>
__device__ __forceinline__ void zero_padding(double* As, double* Bs, int lane) {
    using T = SpreadTile<L>;
    for (int e = lane; e < (8 - L) * T::LDP; e += 32) As[L * T::LDP + e] = 0.0;
    for (int e = lane; e < (T::NT * 8 - T::L2) * T::LDP; e += 32) Bs[T::L2 * T::LDP + e] = 0.0;
}

// Fixed-order pairwise tree over red[0 .. 32 NW), run by the whole CTA (the
// 128-thread tree for NW = 4); ends synchronised, result in red[0].
template <int NW>
__device__ __forceinline__ double block_tree_sum(double* red) {
    constexpr int n = 32 * NW;
    constexpr int top = n > 128 ? 128 : n > 64 ? 64 : n > 32 ? 32 : 16;
    for (int o = top; o > 0; o >>= 1) {
        if (threadIdx.x < o && threadIdx.x + o < n) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    return red[0];
}

// Column epilogue shared by the spread kernels: cross-warp sum of the warps'
// T1 partials (at sm + w * per_warp + t1off, [L^2][RP]), then either the fused
// y, x contractions into this column's partial core (Fpart) or the T1 slab.
// epi: scratch for the contractions (spread_epilogue_doubles), not
// overlapping any warp's T1 partial.
template <int L, int NW = 4>
__device__ __forceinline__ void spread_epilogue(const ColumnArgs& a, const ColumnRange& cr, double* sm,
                                                int per_warp, int t1off, int RP, double* epi,
                                                double* red, double qsum, int want_fwd) {
    constexpr int L2 = L * L, NT_ = 32 * NW;
    const Geometry& g = a.g;
    const int R = g.R;
    __syncthreads();
    red[threadIdx.x] = qsum;
    if (want_fwd && a.Fpart) {
        // Fused y, x contractions: this column segment's partial core
        //   Fcol[r0][r1][r2] = sum_{i,j} W0[r0][x_i] W1[r1][y_j] T1col[(i,j)][r2]
        // (the V_1, V_0 phases of spkmv restricted to one column; summed over
        // columns in order by k_core_sum).
        double* tc = epi;  // [L^2][R]
        double* u = tc + L2 * R;            // [L][R][R]
        __syncthreads();
        for (int e = threadIdx.x; e < L2 * R; e += NT_) {
            const int ij = e / R, r = e % R;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += sm[w * per_warp + t1off + ij * RP + r];
            tc[e] = s;
        }
        __syncthreads();
        double* w01 = u + L * R * R;  // [2][R][L] the column's W0 / W1 rows
        for (int e = threadIdx.x; e < R * L; e += NT_) {
            w01[e] = a.W0[(int64_t)(e / L) * g.n[0] + cr.c0 * L + e % L];
            w01[R * L + e] = a.W1[(int64_t)(e / L) * g.n[1] + cr.c1 * L + e % L];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < L * R * R; e += NT_) {
            const int i = e / (R * R), r1 = (e / R) % R, r2 = e % R;
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < L; ++j) s = fma(w01[R * L + r1 * L + j], tc[(i * L + j) * R + r2], s);
            u[e] = s;
        }
        __syncthreads();
        // Fpart is entry-major, [R^3+1][nblocks], so k_core_sum reads it coalesced
        const int nblocks = a.fstride > 0 ? a.fstride : a.S * g.K[0] * g.K[1];
        double* dst = a.Fpart + (int64_t)cr.seg * g.K[0] * g.K[1] + cr.col;
        for (int e = threadIdx.x; e < R * R * R; e += NT_) {
            const int r0 = e / (R * R), rr = e % (R * R);
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < L; ++i) s = fma(w01[r0 * L + i], u[i * R * R + rr], s);
            dst[(int64_t)e * nblocks] = s;
        }
        __syncthreads();
        const double qs = block_tree_sum<NW>(red);
        if (threadIdx.x == 0) dst[(int64_t)R * R * R * nblocks] = qs;
        return;
    }
    if (want_fwd) {
        double* dst = a.T1 + (int64_t)cr.seg * g.n[0] * g.n[1] * R;
        for (int e = threadIdx.x; e < L2 * R; e += NT_) {
            const int ij = e / R, r = e % R, i = ij / L, j = ij % L;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += sm[w * per_warp + t1off + ij * RP + r];
            dst[((int64_t)(cr.c0 * L + i) * g.n[1] + cr.c1 * L + j) * R + r] = s;
        }
    }
    if (a.colq) {
        __syncthreads();
        const double qs = block_tree_sum<NW>(red);
        if (threadIdx.x == 0) a.colq[(int64_t)cr.seg * g.K[0] * g.K[1] + cr.col] = qs;
    }
}

// The fused epilogue for the common R = 2M + 1 = RC (RC = 9 at M = 4), with
// compile-time index arithmetic, every thread's outputs of a phase in flight
// together, the column's W0 / W1 rows already in shared memory (w01, loaded by
// spread_epilogue_tables at kernel start) and a shuffle tree for sum q.
template <int L>
__device__ __forceinline__ void spread_epilogue_tables(const ColumnArgs& a, const ColumnRange& cr, double* epi,
                                                       int nthreads) {
    const Geometry& g = a.g;
    const int R = g.R;
    double* w01 = epi + L * L * R + L * R * R;  // [2][R][L]
    if (a.Fpart)
        for (int e = threadIdx.x; e < R * L; e += nthreads) {
            w01[e] = a.W0[(int64_t)(e / L) * g.n[0] + cr.c0 * L + e % L];
            w01[R * L + e] = a.W1[(int64_t)(e / L) * g.n[1] + cr.c1 * L + e % L];
        }
}
template <int L, int NW, int RC>
__device__ __forceinline__ void spread_epilogue_rc(const ColumnArgs& a, const ColumnRange& cr, double* sm,
                                                   int per_warp, int t1off, int RP, double* epi,
                                                   double* red, double qsum,
                                                   const double* w01_at = nullptr) {
    constexpr int L2 = L * L, NTH = 32 * NW, RR = RC * RC;
    const Geometry& g = a.g;
    const int tid = threadIdx.x;
    double* tc = epi;                // [L^2][RC]
    double* u = tc + L2 * RC;        // [L][RC][RC]
    const double* w01 = w01_at ? w01_at : u + L * RR;  // [2][RC][L]
    double qs = qsum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, o);
    __syncthreads();  // every warp's T1 partial is in shared memory
    if ((tid & 31) == 0) red[tid >> 5] = qs;
    {
        constexpr int N = L2 * RC, IT = (N + NTH - 1) / NTH;
        double sv[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = min(tid + it * NTH, N - 1), ij = e / RC, r = e % RC;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += sm[w * per_warp + t1off + ij * RP + r];
            sv[it] = s;
        }
#pragma unroll
        for (int it = 0; it < IT; ++it)
            if (tid + it * NTH < N) tc[tid + it * NTH] = sv[it];
    }
    __syncthreads();
    {
        constexpr int N = L * RR, IT = (N + NTH - 1) / NTH;
        double sv[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = min(tid + it * NTH, N - 1), i = e / RR, r1 = (e / RC) % RC, r2 = e % RC;
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < L; ++j) s = fma(w01[RC * L + r1 * L + j], tc[(i * L + j) * RC + r2], s);
            sv[it] = s;
        }
#pragma unroll
        for (int it = 0; it < IT; ++it)
            if (tid + it * NTH < N) u[tid + it * NTH] = sv[it];
    }
    __syncthreads();
    const int nblocks = a.fstride > 0 ? a.fstride : a.S * g.K[0] * g.K[1];
    double* dst = a.Fpart + (int64_t)cr.seg * g.K[0] * g.K[1] + cr.col;
    {
        constexpr int N = RR * RC, IT = (N + NTH - 1) / NTH;
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = tid + it * NTH;
            if (e < N) {
                const int r0 = e / RR, rr = e % RR;
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < L; ++i) s = fma(w01[r0 * L + i], u[i * RR + rr], s);
                dst[(int64_t)e * nblocks] = s;
            }
        }
    }
    if (tid == 0) {
        double q = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) q += red[w];
        dst[(int64_t)RR * RC * nblocks] = q;
    }
}

template <int L, bool MONO>
__global__ void __launch_bounds__(128, SPREAD_MINB) k_spread_mma(ColumnArgs a, int want_fwd) {
    using T = SpreadTile<L>;
    constexpr int L2 = T::L2, L3 = L2 * L, NT = T::NT, LDP = T::LDP, NW = T::NW, CH = T::CH;
    constexpr int MT2 = T::MT2, KS2 = T::KS2, LDK = T::LDK;
    const Geometry& g = a.g;
    const int R = g.R, RT = (R + 7) / 8, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int RP = RT * 8;
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    const int per_warp = spread_warp_doubles<L>(R);
    double* As = sm + warp * per_warp;  // [8][LDP]       q w0, particle-contiguous
    double* Bs = As + 8 * LDP;          // [NT*8][LDP]    w1 (x) w2
    double* ph = As;                    // [MT2*8][LDK]   finished cell grid (aliases staging)
    double* t1w = As + T::stage;        // [MT2*8][RP]    warp partial of T1
    __shared__ double lc[16];
    __shared__ double red[128];
    lagrange_consts(L, lc);
    for (int e = lane; e < MT2 * 8 * RP; e += 32) t1w[e] = 0.0;
    const CellAxis ax0 = cell_axis_tab(a.cellax[0], cr.c0), ax1 = cell_axis_tab(a.cellax[1], cr.c1);
    const int p = lane & (CH - 1), half = CH == 32 ? 0 : lane >> 4;
    double qsum = 0.0;
    zero_padding<L>(As, Bs, lane);
    __syncthreads();

    // Each warp takes a contiguous run of cells holding ~1/NW of the column
    // segment's particles (a deterministic, data-dependent split).
    const int col_cell0 = (cr.c0 * g.K[1] + cr.c1) * g.K[2];
    int zw0, zw1;
    {
        const int P0 = a.start[col_cell0 + cr.zb], P1 = a.start[col_cell0 + cr.ze];
        const int t0 = P0 + (int)((long long)(P1 - P0) * warp / NW);
        const int t1 = P0 + (int)((long long)(P1 - P0) * (warp + 1) / NW);
        zw0 = warp == 0 ? cr.zb
                        : warp_lower_bound(a.start, col_cell0 + cr.zb, col_cell0 + cr.ze, t0, lane) - col_cell0;
        zw1 = warp == NW - 1 ? cr.ze
                             : warp_lower_bound(a.start, col_cell0 + cr.zb, col_cell0 + cr.ze, t1, lane) - col_cell0;
    }
    int s_next = a.start[col_cell0 + zw0];
    for (int c2 = zw0; c2 < zw1; ++c2) {
        const int cell = col_cell0 + c2;
        const int s0 = s_next, s1 = a.start[cell + 1];
        s_next = s1;
        if (s0 == s1) {
            if (a.phi_cells)
                for (int node = lane; node < L3; node += 32) a.phi_cells[(int64_t)cell * L3 + node] = 0.0;
            continue;
        }
        const CellAxis ax2 = cell_axis_tab(a.cellax[2], c2);
        double acc[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
        // lanes past the chunk end clamp to a valid particle and carry q = 0
        double4 nxt = ld_rec(a.sp + s0 + min(p, s1 - s0 - 1));
        for (int base = s0; base < s1; base += CH) {
            const int cnt = min(CH, s1 - base);
            const double4 pt = nxt;  // software prefetch of the next chunk
            if (base + CH < s1) nxt = ld_rec(a.sp + base + CH + min(p, s1 - base - CH - 1));
            double w0[L], w1[L], w2[L];
            const double qv = p < cnt ? pt.w : 0.0;
            qsum += half == 0 ? qv : 0.0;
            if (SPREAD_SKIP & 4) {
#pragma unroll
                for (int k = 0; k < L; ++k) w0[k] = w1[k] = w2[k] = pt.x + k;
            } else if (MONO) {
                powers<L>(ax0.lo, ax0.hi, ax0.mid, ax0.inv, pt.x, w0, a.bad);
                powers<L>(ax1.lo, ax1.hi, ax1.mid, ax1.inv, pt.y, w1, a.bad);
                powers<L>(ax2.lo, ax2.hi, ax2.mid, ax2.inv, pt.z, w2, a.bad);
            } else {
                lagrange_fast<L>(lc, ax0.lo, ax0.hi, ax0.mid, ax0.inv, pt.x, w0, a.bad);
                lagrange_fast<L>(lc, ax1.lo, ax1.hi, ax1.mid, ax1.inv, pt.y, w1, a.bad);
                lagrange_fast<L>(lc, ax2.lo, ax2.hi, ax2.mid, ax2.inv, pt.z, w2, a.bad);
            }
            __syncwarp();
            if (SPREAD_SKIP & 2) {
                As[p] = qv * w0[0] * w1[1] * w2[2];
            } else if constexpr (CH == 32) {
                // one particle per lane: its A row (q w0) and B row (w1 (x) w2)
#pragma unroll
                for (int i = 0; i < L; ++i) As[i * LDP + p] = qv * w0[i];
#pragma unroll
                for (int jj = 0; jj < L; ++jj)
#pragma unroll
                    for (int kk = 0; kk < L; ++kk) Bs[(jj * L + kk) * LDP + p] = w1[jj] * w2[kk];
            } else {
                // lane pair (p, p+16): A rows [4h, 4h+4) and B rows j in [JH h, JH h + JH)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (i < L) {
                        const double lo_w = w0[i], hi_w = (4 + i < L) ? w0[4 + i < L ? 4 + i : 0] : 0.0;
                        As[(half * 4 + i) * LDP + p] = qv * (half ? hi_w : lo_w);  // rows >= L get 0
                    }
                constexpr int JH = (L + 1) / 2;
#pragma unroll
                for (int jj = 0; jj < JH; ++jj) {
                    const double a_lo = w1[jj];
                    const double a_hi = (JH + jj < L) ? w1[JH + jj < L ? JH + jj : 0] : 0.0;
                    const double wj = half ? a_hi : a_lo;
                    const int row = (half * JH + jj) * L;
#pragma unroll
                    for (int kk = 0; kk < L; ++kk) Bs[(row + kk) * LDP + p] = wj * w2[kk];  // rows >= L^2 get 0
                }
            }
            __syncwarp();
            const int ks = (SPREAD_SKIP & 1) ? 0 : (cnt + 3) >> 2;
            for (int kk = 0; kk < ks; ++kk) {
                const int col = kk * 4 + (lane & 3);
                const double af = As[(lane >> 2) * LDP + col];
#pragma unroll
                for (int t = 0; t < NT; ++t) dmma884(acc[t], af, Bs[(t * 8 + (lane >> 2)) * LDP + col]);
            }
        }
        __syncwarp();  // staging reads done: reuse it as ph[(i,j)][k]
        for (int e = lane; e < MT2 * 8 * LDK; e += 32) ph[e] = 0.0;
        __syncwarp();
        const int i_row = lane >> 2;
        if (i_row < L) {
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int col = t * 8 + 2 * (lane & 3) + c;
                    if (col < L2) ph[(i_row * L + col / L) * LDK + col % L] = acc[t][c];
                }
        }
        __syncwarp();
        if (a.phi_cells)
            for (int node = lane; node < L3; node += 32)
                a.phi_cells[(int64_t)cell * L3 + node] = ph[(node / L) * LDK + node % L];
        if (want_fwd && !(SPREAD_SKIP & 8)) {
            // T1c = ph[(i,j)][k] (MT2*8 x LDK) . W2s[k][r] (LDK x RP)
            double bf[KS2][4];
            const double* w2g = a.W2 + c2 * L;
#pragma unroll
            for (int s = 0; s < KS2; ++s)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int k = s * 4 + (lane & 3), r = t * 8 + (lane >> 2);
                    bf[s][t] = (t < RT && k < L && r < R) ? __ldg(w2g + (int64_t)r * g.n[2] + k) : 0.0;
                }
#pragma unroll
            for (int mt = 0; mt < MT2; ++mt) {
                double c[4][2];
#pragma unroll
                for (int t = 0; t < 4; ++t) c[t][0] = c[t][1] = 0.0;
#pragma unroll
                for (int s = 0; s < KS2; ++s) {
                    const double af = ph[(mt * 8 + (lane >> 2)) * LDK + s * 4 + (lane & 3)];
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (t < RT) dmma884(c[t], af, bf[s][t]);
                }
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (t < RT) {
                        double* dst = t1w + (mt * 8 + (lane >> 2)) * RP + t * 8 + 2 * (lane & 3);
                        dst[0] += c[t][0];
                        dst[1] += c[t][1];
                    }
            }
        }
        __syncwarp();
        zero_padding<L>(As, Bs, lane);
        __syncwarp();
    }
    spread_epilogue<L>(a, cr, sm, per_warp, T::stage, RP,
                       spread_epilogue_doubles(L, R) <= T::stage ? sm : sm + NW * per_warp, red,
                       qsum, want_fwd);
}

// Spread, factored-operand variant (monomial basis, L <= 8): the same
// per-cell GEMM phi[i][n] = sum_p (q t0^i)_p B[p][n] over the L^2 pairs
// n = (j, k), with the m8n8k4 B fragment of lane (g = lane/4, p = lane%4) at
// n-tile t factored as B[p][8t + g] = U[p][g] * bv_p^t:
//   g < L:   (j, k) = (g, t),                          U = t1^g,         bv = t2
//   g >= L:  e = (g-L) NT + t, (j, k) = (e%L, NT+e/L),  U = t1^j0 t2^k,   bv = t1
// (the k >= NT pairs; no lane's slots wrap across k for L <= 8, and lanes whose
// only valid slot is t = 0 take bv = 0). Per 16-particle chunk a lane pair
// stages one particle's A row (q t0^i, 8) and U row (8) plus (t1, t2) in
// shared memory -- 18 doubles per particle instead of the 48 of k_spread_mma
// -- and each k-step forms its B fragments in registers (5 DMUL) while the
// tensor pipe runs the DMMAs.
template <int L>
struct UvMap {
    static constexpr int L2 = L * L;
    static constexpr int NT = (L2 + 7) / 8;
    static constexpr int MT2 = (L2 + 7) / 8;
    static constexpr int KS2 = (L + 3) / 4;
    static constexpr int LDK = KS2 * 4 + 4;  // ph row stride: 2 LDK = 8 mod 16 words, conflict-free A reads
    // (j, k) of column n = 8 t + g as j * L + k; -1 for a padding slot
    __host__ __device__ static constexpr int pair(int g, int t) {
        if (t >= NT) return -1;
        if (g < L) return g * L + t;  // k = t < L since NT <= L
        const int e = (g - L) * NT + t;
        const int j = e % L, k = NT + e / L;
        return k < L ? j * L + k : -1;
    }
    // exponents of U for lane group g (U = t1^eu1 t2^eu2; -1: U = 0)
    __host__ __device__ static constexpr int eu1(int g) {
        return g < L ? g : (pair(g, 0) >= 0 ? pair(g, 0) / L : -1);
    }
    __host__ __device__ static constexpr int eu2(int g) {
        return g < L ? 0 : (pair(g, 0) >= 0 ? pair(g, 0) % L : -1);
    }
    // slots t >= 1 valid for group g (else bv = 0)
    __host__ __device__ static constexpr bool multi(int g) { return NT > 1 && pair(g, 1) >= 0; }
    static constexpr int stage = 16 * 8 * 2 + 16 * 2;  // A rows, U rows, (t1, t2)
    static constexpr int ph = MT2 * 8 * LDK;
    static constexpr int area = stage + ph;  // ph separate: its padding is zeroed once
};

// T1 partial row stride (the padded R; shared memory is the occupancy limit).
__host__ __device__ constexpr int uv_t1_stride(int R) { return ((R + 7) / 8) * 8; }

template <int L>
__host__ __device__ constexpr int spread_uv_warp_doubles(int R) {
    return UvMap<L>::area + UvMap<L>::MT2 * 8 * uv_t1_stride(R);
}

// 16-byte-chunk XOR swizzle of an 8-double row: conflict-free 16-lane row
// stores and 32-lane fragment reads.
__device__ __forceinline__ int uv_swz(int row, int col) {
    return row * 8 + ((((col >> 1) ^ (row >> 1)) & 3) << 1) + (col & 1);
}

#ifndef UV_NW
#define UV_NW 4  // warps per column CTA of k_spread_uv
#endif
// CTA shared memory of k_spread_uv: UV_NW warp areas, the column's W2 (R x n2)
// and the epilogue scratch.
template <int L>
__host__ __device__ constexpr size_t spread_uv_smem_doubles(int R, int n2) {
    return UV_NW * (size_t)spread_uv_warp_doubles<L>(R) + (size_t)R * n2 +
           (size_t)spread_epilogue_doubles(L, R);
}

#ifndef UV_SKIP
#define UV_SKIP 0  // profiling ablations only: 1 k-step loop, 2 per-cell drain + contraction,
                   // 4 epilogue, 8 raw per-cell fragments to a scratch buffer, 16 contraction only
#endif
__device__ double* uv_scratch;
// RTM: n-tiles of the W2 contraction held in registers (2: R <= 16, 4: R <= 32).
template <int L, int RTM>
__global__ void __launch_bounds__(32 * UV_NW, SPREAD_MINB) k_spread_uv(ColumnArgs a, int want_fwd) {
    using M = UvMap<L>;
    constexpr int L2 = M::L2, L3 = L2 * L, NT = M::NT, MT2 = M::MT2, KS2 = M::KS2, LDK = M::LDK;
    constexpr int NW = UV_NW, NTH = 32 * NW;
    const Geometry& g = a.g;
    const int R = g.R, RT = (R + 7) / 8, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int RP = uv_t1_stride(R), n2 = g.n[2];
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    const int per_warp = spread_uv_warp_doubles<L>(R);
    double* As = sm + warp * per_warp;  // [16][8] swizzled rows q t0^i
    double* Us = As + 16 * 8;           // [16][8] swizzled rows U
    double2* Ts = reinterpret_cast<double2*>(Us + 16 * 8);  // [16] (t1, t2)
    double* ph = As + M::stage;         // [MT2*8][LDK] finished cell grid
    double* t1w = As + M::area;         // [MT2*8][RP]  warp partial of T1
    double* w2s = sm + NW * per_warp;   // [R][n2] W2 (monomial rows), shared by the CTA
    double* epi = w2s + R * n2;
    __shared__ double red[NTH];
    __shared__ int cst[66];             // cell starts of this column segment (+1)
    for (int e = lane; e < MT2 * 8 * RP; e += 32) t1w[e] = 0.0;
    for (int e = lane; e < M::ph; e += 32) ph[e] = 0.0;  // padding stays zero
    for (int e0 = threadIdx.x; e0 < R * n2; e0 += NTH * 8) {  // loads in flight together
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (e0 + NTH * u < R * n2) v[u] = __ldg(a.W2 + e0 + NTH * u);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (e0 + NTH * u < R * n2) w2s[e0 + NTH * u] = v[u];
    }
    const int col_cell0 = (cr.c0 * g.K[1] + cr.c1) * g.K[2];
    const int nz = cr.ze - cr.zb;
    const bool cst_ok = nz + 1 <= 66;
    if (cst_ok)
        for (int e = threadIdx.x; e <= nz; e += NTH) cst[e] = a.start[col_cell0 + cr.zb + e];
    const CellAxis ax0 = cell_axis_tab(a.cellax[0], cr.c0), ax1 = cell_axis_tab(a.cellax[1], cr.c1);
    // staging role: lane pair (p, h); fragment role: (gg, tg)
    const int p = lane & 15, h = lane >> 4;
    const int gg = lane >> 2, tg = lane & 3;
    const bool use_t2 = gg < L, multi = M::multi(gg);
    double tmax = 0.0;  // largest |t| seen (out-of-cell check at the end)
    double qsum = 0.0;
    // the warp's partial of T1 = sum over its cells of ph_c . W2_c, accumulated
    // by the contraction DMMAs in registers across cells (no per-cell drain)
    double t1acc[MT2][RTM][2];
#pragma unroll
    for (int mt = 0; mt < MT2; ++mt)
#pragma unroll
        for (int t = 0; t < RTM; ++t) t1acc[mt][t][0] = t1acc[mt][t][1] = 0.0;
    __syncthreads();
    auto cstart = [&](int c2) { return cst_ok ? cst[c2 - cr.zb] : a.start[col_cell0 + c2]; };

    // Warp w takes particles [pw0, pw1), an exact quarter of the column
    // segment; its end cells are shared with the neighbouring warps (the
    // contraction is linear, so partial cells simply add). Stage output
    // (phi_cells) needs whole cells: then the split is at cell boundaries.
    int zw0, zw1, pw0, pw1;
    {
        const int P0 = cstart(cr.zb), P1 = cstart(cr.ze);
        const int t0 = P0 + (int)((long long)(P1 - P0) * warp / NW);
        const int t1 = P0 + (int)((long long)(P1 - P0) * (warp + 1) / NW);
        auto lb = [&](int target) {  // first c in [zb, ze] with cstart(c) >= target
            return warp_lower_bound(a.start, col_cell0 + cr.zb, col_cell0 + cr.ze, target, lane) - col_cell0;
        };
        if (a.phi_cells) {
            zw0 = warp == 0 ? cr.zb : lb(t0);
            zw1 = warp == NW - 1 ? cr.ze : lb(t1);
            pw0 = cstart(zw0);
            pw1 = cstart(zw1);
        } else {
            pw0 = t0;
            pw1 = t1;
            zw0 = t0 < t1 ? lb(t0 + 1) - 1 : cr.zb;
            zw1 = t0 < t1 ? lb(t1) : cr.zb;
        }
    }
    for (int c2 = zw0; c2 < zw1; ++c2) {
        const int s0 = max(cstart(c2), pw0), s1 = min(cstart(c2 + 1), pw1);
        if (s0 >= s1) {
            if (a.phi_cells)
                for (int node = lane; node < L3; node += 32)
                    a.phi_cells[(int64_t)(col_cell0 + c2) * L3 + node] = 0.0;
            continue;
        }
        const CellAxis ax2 = cell_axis_tab(a.cellax[2], c2);
        double acc[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
        // lanes past the chunk end clamp to a valid particle and carry q = 0;
        // records of the next two chunks in flight
        double4 nxt = ld_rec(a.sp + min(s0 + p, s1 - 1));
        double4 nxt2 = ld_rec(a.sp + min(s0 + 16 + p, s1 - 1));
        for (int base = s0; base < s1; base += 16) {
            const int cnt = min(16, s1 - base);
            const double4 pt = nxt;
            nxt = nxt2;
            if (base + 32 < s1) nxt2 = ld_rec(a.sp + min(base + 32 + p, s1 - 1));
            const double q = p < cnt ? pt.w : 0.0;
            qsum += h == 0 ? q : 0.0;
            const double t0 = (pt.x - ax0.mid) * ax0.inv;
            const double t1 = (pt.y - ax1.mid) * ax1.inv;
            const double t2 = (pt.z - ax2.mid) * ax2.inv;
            tmax = fmax(tmax, fmax(fabs(t0), fmax(fabs(t1), fabs(t2))));
            __syncwarp();  // previous chunk's fragment reads done
            double row[8];
            if (h == 0) {
                double w = q;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    row[i] = i < L ? w : 0.0;
                    w *= t0;
                }
            } else {
                double p1[L], p2[L];
                p1[0] = p2[0] = 1.0;
#pragma unroll
                for (int e = 1; e < L; ++e) {
                    p1[e] = p1[e - 1] * t1;
                    p2[e] = p2[e - 1] * t2;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int e1 = M::eu1(i), e2 = M::eu2(i);
                    row[i] = e1 < 0 ? 0.0 : (e2 == 0 ? p1[e1 < 0 ? 0 : e1] : p1[e1 < 0 ? 0 : e1] * p2[e2 < 0 ? 0 : e2]);
                }
                Ts[p] = make_double2(t1, t2);
            }
            double* dst = h == 0 ? As : Us;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<double2*>(dst + uv_swz(p, 2 * c)) = make_double2(row[2 * c], row[2 * c + 1]);
            __syncwarp();
            const int ks = (UV_SKIP & 1) ? 0 : (cnt + 3) >> 2;
            for (int kk = 0; kk < ks; ++kk) {
                const int r = kk * 4 + tg;
                const double2 tt = Ts[r];
                const double af = As[uv_swz(r, gg)];
                const double u = Us[uv_swz(r, gg)];
                const double bv = multi ? (use_t2 ? tt.y : tt.x) : 0.0;
                double v[NT];
                v[0] = u;
#pragma unroll
                for (int t = 1; t < NT; ++t) v[t] = v[t - 1] * bv;
#pragma unroll
                for (int t = 0; t < NT; ++t) dmma884(acc[t], af, v[t]);
            }
        }
        __syncwarp();
        if (UV_SKIP & 8) {  // ablation: raw fragments straight to global
            double2* o = reinterpret_cast<double2*>(uv_scratch) + ((int64_t)(col_cell0 + c2) * NT) * 32 + lane;
#pragma unroll
            for (int t = 0; t < NT; ++t) o[t * 32] = make_double2(acc[t][0], acc[t][1]);
        }
        if (UV_SKIP & 2) continue;
        const int i_row = lane >> 2;
        if (i_row < L) {
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int jk = M::pair(2 * (lane & 3) + c, t);
                    if (jk >= 0) ph[(i_row * L + jk / L) * LDK + jk % L] = acc[t][c];
                }
        }
        __syncwarp();
        if (a.phi_cells)
            for (int node = lane; node < L3; node += 32)
                a.phi_cells[(int64_t)(col_cell0 + c2) * L3 + node] = ph[(node / L) * LDK + node % L];
        if (want_fwd && !(UV_SKIP & 16)) {
            // T1c = ph[(i,j)][k] (MT2*8 x LDK) . W2s[k][r] (LDK x RP)
            double bf[KS2][4];
            const double* w2c = w2s + c2 * L;
#pragma unroll
            for (int s = 0; s < KS2; ++s)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int k = s * 4 + (lane & 3), rr = t * 8 + (lane >> 2);
                    bf[s][t] = (t < RT && k < L && rr < R) ? w2c[rr * n2 + k] : 0.0;
                }
#pragma unroll
            for (int mt = 0; mt < MT2; ++mt)
#pragma unroll
                for (int s = 0; s < KS2; ++s) {
                    const double af = ph[(mt * 8 + (lane >> 2)) * LDK + s * 4 + (lane & 3)];
#pragma unroll
                    for (int t = 0; t < RTM; ++t)
                        if (t < RT) dmma884(t1acc[mt][t], af, bf[s][t]);
                }
        }
        __syncwarp();
    }
    if (want_fwd) {
#pragma unroll
        for (int mt = 0; mt < MT2; ++mt)
#pragma unroll
            for (int t = 0; t < RTM; ++t)
                if (t < RT)
                    *reinterpret_cast<double2*>(t1w + (mt * 8 + (lane >> 2)) * RP + t * 8 + 2 * (lane & 3)) =
                        make_double2(t1acc[mt][t][0], t1acc[mt][t][1]);
        __syncwarp();
    }
    // tensor_weights' out-of-cell check, |t| <= 1 + 2e-12 (slack 1e-12 of the width)
    const unsigned badw = __ballot_sync(0xffffffffu, !(tmax <= 1.0 + 2e-12));
    if (lane == 0 && badw) atomicOr(&a.bad[1], 1ull);
    if (UV_SKIP & 4) return;
    spread_epilogue<L, NW>(a, cr, sm, per_warp, M::area, RP, epi, red, qsum, want_fwd);
}

// ---------------------------------------------------------------------------
// Spread, split-exponent variant (monomial basis, L = 4 and 6). With m = L/2
// and every exponent split as e = m e_hi + e_lo (e_hi in {0,1}, e_lo < m),
//     t0^i t1^j t2^k = [t0^(m ih) t1^(m jh) t2^(m kh)] * [t0^il t1^jl t2^kl],
// so the cell's L^3 grid is ONE (8 x m^3) = (8 x P)(P x m^3) GEMM:
//     row g = (ih, jh, kh)  A[g][p]   = q_p T0^ih T1^jh T2^kh  (T = t^m)
//     col   = (il, jl, kl)  B[p][col] = t0^il t1^jl t2^kl
// No padded rows (the (L x L^2) form wastes 2 of 8 rows at L = 6) and 27 of
// 32 columns used at L = 6 (all 8 at L = 4): 4 DMMAs per k-step instead of 5.
// One particle per lane stages its row (no divergent half-warp paths); at
// L = 6 the B fragment of lane group g at n-tile t < 3 is U_g t0^t with
// U_g = t1^jl t2^kl over (jl, kl) = (g / 3, g % 3), and tile 3 holds the
// three (il, 2, 2) columns as W[g] = t0^g t1^2 t2^2.
#ifndef F8_SKIP
#define F8_SKIP 0  // profiling ablations only: 1 k-steps, 2 per-cell drain + contraction, 4 epilogue, 8 staging
#endif
#ifndef F8_NW
#define F8_NW 4  // warps per column CTA of the split-exponent spread
#endif
#ifndef F8_RING
#define F8_RING 2
#endif
__device__ __forceinline__ void cp_async16_sm(void* dst, const void* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_sm(void* dst, const void* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int L>
struct F8Map {
    static_assert(L == 4 || L == 6, "split-exponent spread: L = 4 or 6");
    static constexpr int m = L / 2;
    static constexpr int NT = L == 6 ? 4 : 1;
    static constexpr int SR = 20;              // staged row stride (conflict-free LDS.128)
    static constexpr int L2 = L * L;
    static constexpr int MT2 = (L2 + 7) / 8;
    static constexpr int KS2 = (L + 3) / 4;
    static constexpr int LDK = KS2 * 4 + 4;
    static constexpr int stage = 32 * SR;      // also the warp's T1 partial at the end
    static constexpr int ph = MT2 * 8 * LDK;
    static constexpr int RING = F8_RING;       // chunks of particle records in flight (cp.async)
    static constexpr int area = stage + ph + RING * 32 * 4;
    // grid node (i, j, k) of accumulator column `col` at row group g
    __device__ static int node(int g, int col) {
        const int ih = (g >> 2) & 1, jh = (g >> 1) & 1, kh = g & 1;
        int il, jl, kl;
        if (L == 6) {
            const int t = col >> 3, c = col & 7;
            if (t < 3) {
                il = t;
                jl = c / 3;
                kl = c % 3;
            } else {
                if (c >= 3) return -1;
                il = c;
                jl = kl = 2;
            }
        } else {
            il = (col >> 2) & 1;
            jl = (col >> 1) & 1;
            kl = col & 1;
        }
        const int i = m * ih + il, j = m * jh + jl, k = m * kh + kl;
        return (i * L + j) * L + k;
    }
};

// The warp's T1 partial [MT2*8][RP] reuses the staging rows after the last
// chunk (MT2*8*RP <= 32*SR for R <= 16; larger R appends it).
template <int L>
__host__ __device__ constexpr int spread_f8_t1off(int R) {
    return F8Map<L>::MT2 * 8 * uv_t1_stride(R) <= F8Map<L>::stage ? 0 : F8Map<L>::area;
}
template <int L>
__host__ __device__ constexpr int spread_f8_warp_doubles(int R) {
    return F8Map<L>::area + (spread_f8_t1off<L>(R) ? F8Map<L>::MT2 * 8 * uv_t1_stride(R) : 0);
}
template <int L>
__host__ __device__ constexpr size_t spread_f8_smem_doubles(int R, int /*n2*/) {
    return F8_NW * (size_t)spread_f8_warp_doubles<L>(R) + (size_t)spread_epilogue_doubles(L, R);
}

// MINB: CTAs per SM the register allocation is sized for. 3 (162 registers)
// when the column CTAs make about one wave at three per SM (config 3: 441
// columns, 45.2 vs 47.6 us at 4); 4 (128 registers, a few spilled bytes) for
// grids of several waves (config 4: 1849 columns, 173.5 vs 179.8 us).
template <int L, int RTM, int MINB>
__global__ void __launch_bounds__(32 * F8_NW, MINB) k_spread_f8(ColumnArgs a, int want_fwd) {
    using M = F8Map<L>;
    constexpr int L3 = L * L * L, NT = M::NT, MT2 = M::MT2, KS2 = M::KS2, LDK = M::LDK, SR = M::SR;
    constexpr int NW = F8_NW, NTH = 32 * F8_NW;
    const Geometry& g = a.g;
    // The monomial W2's row r = 0 is exactly (1, 0, ..., 0) in every cell (k_factor_wl), so
    // T1[(i,j)][0] is the k = 0 entry of the cell grid: the W2 contraction runs over
    // r = 1 .. R-1 (R = 9: one n-tile instead of two) and r = 0 is a running sum.
    const int R = g.R, RT = (R - 1 + 7) / 8, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int RP = uv_t1_stride(R), n2 = g.n[2];
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    TRACE_MARK(0, 0);
    pdl_trigger();  // the core sum's CTAs may take the slots this kernel's CTAs free
    pdl_wait();     // the sort's cell starts and records
    const int per_warp = spread_f8_warp_doubles<L>(R);
    double* St = sm + warp * per_warp;  // [32][SR] staged particle rows
    double* ph = St + M::stage;         // [MT2*8][LDK] finished cell grid
    // [RING][2][32] records, lane-private: (x, y) of the 32 lanes, then (z, q): every 16-byte
    // copy of a warp lands on 512 contiguous bytes (a double4 per lane is 8-way conflicted)
    double2* ring = reinterpret_cast<double2*>(ph + M::ph);
    const int t1off = spread_f8_t1off<L>(R);
    double* t1w = St + t1off;           // [MT2*8][RP]  warp partial of T1 (after the chunks)
    double* epi = sm + NW * per_warp;   // epilogue scratch
    __shared__ double red[NTH];
    __shared__ int cst[66];
    spread_epilogue_tables<L>(a, cr, epi, NTH);  // W0 / W1 column rows, used after the particles
    for (int e = lane; e < M::ph; e += 32) ph[e] = 0.0;  // padding stays zero
    const int col_cell0 = (cr.c0 * g.K[1] + cr.c1) * g.K[2];
    const int nz = cr.ze - cr.zb;
    const bool cst_ok = nz + 1 <= 66;
    if (cst_ok)
        for (int e = threadIdx.x; e <= nz; e += NTH) cst[e] = a.start[col_cell0 + cr.zb + e];
    const CellAxis ax0 = cell_axis_tab(a.cellax[0], cr.c0), ax1 = cell_axis_tab(a.cellax[1], cr.c1);
    const int gg = lane >> 2, tg = lane & 3;
    double tmax = 0.0, qsum = 0.0;
    double t1acc[MT2][RTM][2];
    constexpr int NR0 = (MT2 * 8 + 31) / 32;
    double t1r0[NR0];
#pragma unroll
    for (int u = 0; u < NR0; ++u) t1r0[u] = 0.0;
#pragma unroll
    for (int mt = 0; mt < MT2; ++mt)
#pragma unroll
        for (int t = 0; t < RTM; ++t) t1acc[mt][t][0] = t1acc[mt][t][1] = 0.0;
    __syncthreads();
    // the column's cell starts: explicit shared-memory loads (through the lambdas
    // the table would be read with generic loads and a window-address rebuild)
    const unsigned cst_sa = (unsigned)__cvta_generic_to_shared(cst);
    const int zb0 = cr.zb;
    const int32_t* gstart = a.start + col_cell0;
    auto cstart = [=](int c2) {
        int v;
        if (cst_ok)
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(cst_sa + 4u * (unsigned)(c2 - zb0)));
        else
            v = gstart[c2];
        return v;
    };

    // Warp w takes particles [pw0, pw1), an exact quarter of the column segment
    // (cells shared by two warps add linearly); whole cells for phi_cells.
    int zw0, zw1, pw0, pw1;
    {
        const int P0 = cstart(cr.zb), P1 = cstart(cr.ze);
        const int t0 = P0 + (int)((long long)(P1 - P0) * warp / NW);
        const int t1 = P0 + (int)((long long)(P1 - P0) * (warp + 1) / NW);
        auto lb = [&](int target) {
            return warp_lower_bound(a.start, col_cell0 + cr.zb, col_cell0 + cr.ze, target, lane) - col_cell0;
        };
        if (a.phi_cells) {
            zw0 = warp == 0 ? cr.zb : lb(t0);
            zw1 = warp == NW - 1 ? cr.ze : lb(t1);
            pw0 = cstart(zw0);
            pw1 = cstart(zw1);
        } else {
            pw0 = t0;
            pw1 = t1;
            zw0 = t0 < t1 ? lb(t0 + 1) - 1 : cr.zb;
            zw1 = t0 < t1 ? lb(t1) : cr.zb;
        }
    }
    // Particle records stream through a lane-private cp.async ring: the
    // producer cursor runs RING - 1 chunks ahead of the consumer over the
    // warp's cell-aligned chunk sequence, across cell boundaries (lane l
    // copies record l of each chunk; lanes past a chunk's end copy its last
    // record: finite t, q masked to 0 below).
    auto cell_lo_p = [&](int c) { return max(cstart(c), pw0); };
    auto cell_hi_p = [&](int c) { return min(cstart(c + 1), pw1); };
    // producer cursor: cell nc2, next record nbase, the cell's end nhi (the
    // table is read only when the cursor enters a cell; empty cells are skipped)
    int nc2 = zw0, nbase = 0, nhi = 0;
    auto enter_cell = [&]() {
        while (nc2 < zw1) {
            nbase = cell_lo_p(nc2);
            nhi = cell_hi_p(nc2);
            if (nbase < nhi) break;
            ++nc2;
        }
    };
    enter_cell();
    int pslot = 0, cslot = 0;
    // direct records: the particle index of the chunk to be issued is loaded
    // one chunk earlier (pidx), so the copies never wait on the perm load
    int pidx = 0;
    auto perm_at = [&]() {
        return nc2 < zw1 ? __ldg(a.perm + min(nbase + lane, nhi - 1)) : 0;
    };
    if (a.direct) pidx = perm_at();
    auto issue = [&]() {
        if (nc2 < zw1) {
            double2* dlo = ring + pslot * 64 + lane;
            double2* dhi = dlo + 32;
            if (a.direct) {
                const double* src = a.xyz + 3 * (int64_t)pidx;
                cp_async8_sm(dlo, src);
                cp_async8_sm(reinterpret_cast<char*>(dlo) + 8, src + 1);
                cp_async8_sm(dhi, src + 2);
                cp_async8_sm(reinterpret_cast<char*>(dhi) + 8, a.qv + pidx);
            } else {
                const double4* src = a.sp + min(nbase + lane, nhi - 1);
                cp_async16_sm(dlo, src);
                cp_async16_sm(dhi, reinterpret_cast<const char*>(src) + 16);
            }
            nbase += 32;
            if (nbase >= nhi) {
                ++nc2;
                enter_cell();
            }
            if (a.direct) pidx = perm_at();
        }
        cp_async_commit();
        pslot = pslot + 1 == M::RING ? 0 : pslot + 1;
    };
    TRACE_MARK(0, 1);
#pragma unroll
    for (int u = 0; u < M::RING - 1; ++u) issue();
    TRACE_DECL(tr_wait);
    TRACE_DECL(tr_issue);
    TRACE_DECL(tr_stage);
    TRACE_DECL(tr_kloop);
    TRACE_DECL(tr_drain);
    for (int c2 = zw0; c2 < zw1; ++c2) {
        const int s0 = cell_lo_p(c2), s1 = cell_hi_p(c2);
        if (s0 >= s1) {
            if (a.phi_cells)
                for (int node = lane; node < L3; node += 32)
                    a.phi_cells[(int64_t)(col_cell0 + c2) * L3 + node] = 0.0;
            continue;
        }
        const CellAxis ax2 = cell_axis_tab(a.cellax[2], c2);
        double acc[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
        for (int base = s0; base < s1; base += 32) {
            const int cnt = min(32, s1 - base);
            TRACE_CLK(c0);
            issue();
            TRACE_CLK(c0b);
            cp_async_wait<M::RING - 1>();
            TRACE_CLK(c1);
            TRACE_ACC(tr_issue, c0, c0b);
            const double2 pxy = ring[cslot * 64 + lane], pzq = ring[cslot * 64 + 32 + lane];
            const double4 pt = make_double4(pxy.x, pxy.y, pzq.x, pzq.y);
            cslot = cslot + 1 == M::RING ? 0 : cslot + 1;
            const double q = lane < cnt ? pt.w : 0.0;
            qsum += q;
            const double t0 = (pt.x - ax0.mid) * ax0.inv;
            const double t1 = (pt.y - ax1.mid) * ax1.inv;
            const double t2 = (pt.z - ax2.mid) * ax2.inv;
            tmax = fmax(tmax, fmax(fabs(t0), fmax(fabs(t1), fabs(t2))));
            __syncwarp();  // previous chunk's fragment reads done
            double* row = St + lane * SR;
            if (F8_SKIP & 8) {
                row[0] = t0 + t1 + t2 + q;
            } else if (L == 6) {
                const double a2 = t0 * t0, b2 = t1 * t1, c2v = t2 * t2;
                const double T0 = a2 * t0, T1 = b2 * t1, T2 = c2v * t2;
                const double qT1 = q * T1, qT0 = q * T0, qT0T1 = qT0 * T1;
                const double b1c1 = t1 * t2, b1c2 = t1 * c2v, b2c1 = b2 * t2, b2c2 = b2 * c2v;
                // [A_g, U_g] pairs, g = (ih, jh, kh) for A and 3 jl + kl for U
                // pair g of row l sits at pair slot (g + ((l >> 2) & 1)) & 7: with the 160-byte
                // row stride, lanes l and l + 4 of a quarter-warp then store to different banks
                // (conflict-free 128-bit stores); a k-step reads rows 4 kk + tg, so its
                // rotation kk & 1 is warp-uniform and the reads stay conflict-free
                const int sh = (lane >> 2) & 1;
                *reinterpret_cast<double2*>(row + 2 * ((0 + sh) & 7)) = make_double2(q, 1.0);
                *reinterpret_cast<double2*>(row + 2 * ((1 + sh) & 7)) = make_double2(q * T2, t2);
                *reinterpret_cast<double2*>(row + 2 * ((2 + sh) & 7)) = make_double2(qT1, c2v);
                *reinterpret_cast<double2*>(row + 2 * ((3 + sh) & 7)) = make_double2(qT1 * T2, t1);
                *reinterpret_cast<double2*>(row + 2 * ((4 + sh) & 7)) = make_double2(qT0, b1c1);
                *reinterpret_cast<double2*>(row + 2 * ((5 + sh) & 7)) = make_double2(qT0 * T2, b1c2);
                *reinterpret_cast<double2*>(row + 2 * ((6 + sh) & 7)) = make_double2(qT0T1, b2);
                *reinterpret_cast<double2*>(row + 2 * ((7 + sh) & 7)) = make_double2(qT0T1 * T2, b2c1);
                // [t0, W0, W1, W2] with W_g = t0^g t1^2 t2^2; the two pairs swap on rotated rows
                *reinterpret_cast<double2*>(row + 16 + 2 * sh) = make_double2(t0, b2c2);
                *reinterpret_cast<double2*>(row + 18 - 2 * sh) = make_double2(b2c2 * t0, b2c2 * a2);
            } else {
                // L = 4: [A_g, B_g], A_g = q t0^(2ih) t1^(2jh) t2^(2kh), B_g = t0^il t1^jl t2^kl
                const double a2 = t0 * t0, b2 = t1 * t1, c2v = t2 * t2;
                const double qb = q * b2, qa = q * a2, qab = qa * b2;
                const double b1c1 = t1 * t2;
                const int sh = (lane >> 2) & 1;  // see L = 6
                *reinterpret_cast<double2*>(row + 2 * ((0 + sh) & 7)) = make_double2(q, 1.0);
                *reinterpret_cast<double2*>(row + 2 * ((1 + sh) & 7)) = make_double2(q * c2v, t2);
                *reinterpret_cast<double2*>(row + 2 * ((2 + sh) & 7)) = make_double2(qb, t1);
                *reinterpret_cast<double2*>(row + 2 * ((3 + sh) & 7)) = make_double2(qb * c2v, b1c1);
                *reinterpret_cast<double2*>(row + 2 * ((4 + sh) & 7)) = make_double2(qa, t0);
                *reinterpret_cast<double2*>(row + 2 * ((5 + sh) & 7)) = make_double2(qa * c2v, t0 * t2);
                *reinterpret_cast<double2*>(row + 2 * ((6 + sh) & 7)) = make_double2(qab, t0 * t1);
                *reinterpret_cast<double2*>(row + 2 * ((7 + sh) & 7)) = make_double2(qab * c2v, t0 * b1c1);
            }
            __syncwarp();
            TRACE_CLK(c2_);
            const int ks = (F8_SKIP & 1) ? 0 : (cnt + 3) >> 2;
            for (int kk = 0; kk < ks; ++kk) {
                const double* r = St + (kk * 4 + tg) * SR;
                const double2 au = *reinterpret_cast<const double2*>(r + 2 * ((gg + (kk & 1)) & 7));
                if (L == 6) {
                    const int s2 = 2 * (kk & 1);  // the row's rotation
                    const double tt = r[16 + s2];
                    const double w = gg < 3 ? r[16 + ((1 + gg + s2) & 3)] : 0.0;
                    const double b1 = au.y * tt;
                    dmma884(acc[0], au.x, au.y);
                    dmma884(acc[3], au.x, w);
                    dmma884(acc[1], au.x, b1);
                    dmma884(acc[2], au.x, b1 * tt);
                } else {
                    dmma884(acc[0], au.x, au.y);
                }
            }
            TRACE_CLK(c3);
            TRACE_ACC(tr_wait, c0, c1);
            TRACE_ACC(tr_stage, c1, c2_);
            TRACE_ACC(tr_kloop, c2_, c3);
        }
        TRACE_CLK(d0);
        __syncwarp();
        if (F8_SKIP & 2) {
            t1acc[0][0][0] += acc[0][0] + acc[NT - 1][1] + St[lane];
            continue;
        }
        // accumulator (g, 8t + 2c + e) -> ph[(i, j)][k]
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int nd = M::node(gg, 8 * t + 2 * tg + e);
                if (nd >= 0) ph[(nd / L) * LDK + nd % L] = acc[t][e];
            }
        __syncwarp();
        if (a.phi_cells)
            for (int node = lane; node < L3; node += 32)
                a.phi_cells[(int64_t)(col_cell0 + c2) * L3 + node] = ph[(node / L) * LDK + node % L];
        if (want_fwd) {
            // T1c = ph[(i,j)][k] (MT2*8 x LDK) . W2s[k][r] (LDK x RP)
            double bf[KS2][4];
            const double* w2c = a.W2 + c2 * L;  // the cell's W2 slice (L1/L2 resident)
#pragma unroll
            for (int s = 0; s < KS2; ++s)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int k = s * 4 + (lane & 3), rr = 1 + t * 8 + (lane >> 2);
                    bf[s][t] = (t < RT && k < L && rr < R) ? __ldg(w2c + (int64_t)rr * n2 + k) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < NR0; ++u)
                if (lane + 32 * u < MT2 * 8) t1r0[u] += ph[(lane + 32 * u) * LDK];
#pragma unroll
            for (int mt = 0; mt < MT2; ++mt)
#pragma unroll
                for (int s = 0; s < KS2; ++s) {
                    const double af = ph[(mt * 8 + (lane >> 2)) * LDK + s * 4 + (lane & 3)];
#pragma unroll
                    for (int t = 0; t < RTM; ++t)
                        if (t < RT) dmma884(t1acc[mt][t], af, bf[s][t]);
                }
        }
        __syncwarp();
        TRACE_CLK(d1);
        TRACE_ACC(tr_drain, d0, d1);
    }
    TRACE_PUT(0, 4, tr_wait);
    TRACE_PUT(0, 8, tr_issue);
    TRACE_PUT(0, 5, tr_stage);
    TRACE_PUT(0, 6, tr_kloop);
    TRACE_PUT(0, 7, tr_drain);
    cp_async_wait<0>();
    __syncwarp();
    TRACE_MARK(0, 2);
    if (want_fwd) {
        // the rows past MT2*8 stay zero: the epilogue reads only (i, j) < L^2
#pragma unroll
        for (int mt = 0; mt < MT2; ++mt)
#pragma unroll
            for (int t = 0; t < RTM; ++t)
                if (t < RT) {
                    const int r = 1 + t * 8 + 2 * (lane & 3);
                    double* dst = t1w + (mt * 8 + (lane >> 2)) * RP;
                    if (r < R) dst[r] = t1acc[mt][t][0];
                    if (r + 1 < R) dst[r + 1] = t1acc[mt][t][1];
                }
#pragma unroll
        for (int u = 0; u < NR0; ++u)
            if (lane + 32 * u < MT2 * 8) t1w[(lane + 32 * u) * RP] = t1r0[u];
        __syncwarp();
    }
    // tensor_weights' out-of-cell check, |t| <= 1 + 2e-12 (slack 1e-12 of the width)
    const unsigned badw = __ballot_sync(0xffffffffu, !(tmax <= 1.0 + 2e-12));
    if (lane == 0 && badw) atomicOr(&a.bad[1], 1ull);
    if (F8_SKIP & 4) {
        if (a.Fpart && sm[threadIdx.x] + qsum == 1.2345) a.Fpart[0] = 0.0;
        return;
    }
    if (want_fwd && a.Fpart && R == 9)
        spread_epilogue_rc<L, NW, 9>(a, cr, sm, per_warp, t1off, RP, epi, red, qsum);
    else
        spread_epilogue<L, NW>(a, cr, sm, per_warp, t1off, RP, epi, red, qsum, want_fwd);
    TRACE_MARK(0, 3);
}

// Records s, s + stride, ... of the sorted order for one gather thread: the
// record one step ahead and its particle index two steps ahead (with direct
// records the record load needs the index; the gather needs no charge).
struct RecStream {
    const ColumnArgs* a;
    int s1, stride;
    double4 nr;
    int ni, nni;
    __device__ double4 fetch(int s, int i) const {
        if (s >= s1) return make_double4(0.0, 0.0, 0.0, 0.0);
        if (a->direct) {
            const double* x = a->xyz + 3 * (int64_t)i;
            return make_double4(__ldg(x), __ldg(x + 1), __ldg(x + 2), 0.0);
        }
        return ld_rec(a->sp + s);
    }
    __device__ int index(int s) const { return s < s1 ? __ldg(a->perm + s) : 0; }
    __device__ void init(int s) {
        ni = index(s);
        nni = index(s + stride);
        nr = fetch(s, ni);
    }
    // record and particle index of s (the stream's next element)
    __device__ double4 next(int s, int& idx) {
        const double4 r = nr;
        idx = ni;
        nr = fetch(s + stride, nni);
        ni = nni;
        nni = index(s + 2 * stride);
        return r;
    }
};

// Backward z-expansion + gather with compile-time L: psi for a batch of the
// column's cells in shared memory, then one thread per particle,
// z = sum_i w0[i] sum_j w1[j] sum_k w2[k] psi[i][j][k] - c_Lambda sum(q),
// scattered straight to global particle order.
#ifndef GATHER_GT
#define GATHER_GT 128
#endif
constexpr int GT = GATHER_GT;  // gather threads per CTA

constexpr int kGatherTab = 32;  // batch cells with shared-memory start/axis tables
template <int L, int MODE, bool MONO>
#ifndef GATHER_SKIP
#define GATHER_SKIP 0  // profiling ablations only: 1 particle loop, 2 Horner
#endif
#ifndef GATHER_PAIRS
#define GATHER_PAIRS 1  // allow two adjacent particles per thread (ColumnArgs::gpairs)
#endif
#ifndef GATHER_MINB
#define GATHER_MINB (512 / GT)
#endif
__global__ void __launch_bounds__(GT, GATHER_MINB) k_bwd_gather_t(ColumnArgs a, int cells_per_batch) {
    constexpr int L2 = L * L, L3 = L2 * L;
    const Geometry& g = a.g;
    const int R = g.R, tid = threadIdx.x;
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    double* b2s = sm;             // L^2 x R
    double* psi = b2s + L2 * R;   // cells_per_batch x L^3
    TRACE_MARK(1, 0);
    __shared__ double lc[16];
    __shared__ int gcst[kGatherTab + 1];
    __shared__ double4 gax[kGatherTab];
    lagrange_consts(L, lc);
    double corr = a.corr ? *a.corr : 0.0;
    if (MODE != GATHER_FROM_CELLS && a.B2 == nullptr) {
        // Fused backward y, x expansions (the U_0, U_1 phases of spkmv) for
        // this column: b2s[(i,j)][r2] = sum_{r0,r1} W0[r0][x_i] W1[r1][y_j] (G .* F)[r0,r1,r2]
        const int RR = R * R;
        double* h = psi + (size_t)cells_per_batch * L3;  // [R^3]  G .* F
        double* v = h + RR * R;                          // [L][R][R]
        double* w01 = v + L * RR;                        // [2][R][L] W0, W1 column rows
        for (int e0 = tid; e0 < RR * R; e0 += GT * 8) {  // loads in flight together
            double gv[8], fv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (e0 + GT * u < RR * R) {
                    gv[u] = __ldg(a.Gc + e0 + GT * u);
                    fv[u] = __ldg(a.Fc + e0 + GT * u);
                }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (e0 + GT * u < RR * R) h[e0 + GT * u] = gv[u] * fv[u];
        }
        if (MONO && tid == 0) {
            // Zero mode, exactly: the m = 0 rows of W_a are the constant 1 and
            // Lagrange interpolation reproduces constants, so F[0,0,0] = sum q
            // and (W^T (G .* F))[0] - c sum q = (G[0] - c) sum q. Evaluated
            // this way, not as the difference of two rounded sums over all
            // particles, which for a neutral system leaves a uniform offset
            // of pure rounding noise ("zero mode").
            h[0] = (__ldg(a.Gc) - a.correction) * __ldg(a.Fc + RR * R);
        }
        for (int e = tid; e < R * L; e += GT) {
            w01[e] = a.W0[(int64_t)(e / L) * g.n[0] + cr.c0 * L + e % L];
            w01[R * L + e] = a.W1[(int64_t)(e / L) * g.n[1] + cr.c1 * L + e % L];
        }
        __syncthreads();
        for (int e = tid; e < L * RR; e += GT) {
            const int i = e / RR, rr = e % RR;
            double s = 0.0;
            for (int r0 = 0; r0 < R; ++r0) s = fma(w01[r0 * L + i], h[r0 * RR + rr], s);
            v[e] = s;
        }
        __syncthreads();
        for (int e = tid; e < L2 * R; e += GT) {
            const int ij = e / R, r2 = e % R, i = ij / L, j = ij % L;
            double s = 0.0;
            for (int r1 = 0; r1 < R; ++r1) s = fma(w01[R * L + r1 * L + j], v[i * RR + r1 * R + r2], s);
            b2s[e] = s;
        }
        corr = MONO ? 0.0 : a.correction * a.Fc[RR * R];
    } else if (MODE != GATHER_FROM_CELLS) {
        for (int e = tid; e < L2 * R; e += GT) {
            const int ij = e / R, r = e % R, i = ij / L, j = ij % L;
            b2s[e] = a.B2[((int64_t)(cr.c0 * L + i) * g.n[1] + cr.c1 * L + j) * R + r];
        }
    }
    const CellAxis ax0 = cell_axis_tab(a.cellax[0], cr.c0), ax1 = cell_axis_tab(a.cellax[1], cr.c1);
    __syncthreads();
    TRACE_MARK(1, 1);
    double* w2s = psi + (size_t)cells_per_batch * L3 + (size_t)R * R * R + (size_t)L * R * R +
                  2 * (size_t)R * L;  // [R][cells_per_batch * L] W2 slice of the batch
    for (int cb0 = cr.zb; cb0 < cr.ze; cb0 += cells_per_batch) {
        const int cb1 = min(cr.ze, cb0 + cells_per_batch);
        const int cell0 = (cr.c0 * g.K[1] + cr.c1) * g.K[2] + cb0;
        const int nz = (cb1 - cb0) * L;
        if (MODE != GATHER_FROM_CELLS) {
            for (int e0 = tid; e0 < R * nz; e0 += GT * 8) {  // loads in flight together
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = e0 + GT * u;
                    if (e < R * nz) v[u] = __ldg(a.W2 + (int64_t)(e / nz) * g.n[2] + cb0 * L + e % nz);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (e0 + GT * u < R * nz) w2s[e0 + GT * u] = v[u];
            }
            __syncthreads();
        }
        if (MODE == GATHER_FROM_CELLS) {
            for (int e = tid; e < (cb1 - cb0) * L3; e += GT)
                psi[e] = a.psi_cells[(int64_t)(cell0 + (e / L3)) * L3 + e % L3];
        } else if (L <= 8 && R <= 16) {
            // psi_cell[(i,j)][k] = sum_r B2col[(i,j)][r] W2[r][c2 L + k]: an
            // (L^2 x R)(R x L) GEMM per cell on DMMA; the B2col fragments stay
            // in registers for all cells of the column.
            constexpr int MT = (L2 + 7) / 8;
            const int warp = tid >> 5, lane = tid & 31;
            constexpr int KSMAX = 4;  // R <= 16
            const int KS = (R + 3) / 4;
            double af[MT][KSMAX];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int ks = 0; ks < KSMAX; ++ks) {
                    const int row = mt * 8 + (lane >> 2), r = ks * 4 + (lane & 3);
                    af[mt][ks] = (ks < KS && row < L2 && r < R) ? b2s[row * R + r] : 0.0;
                }
            for (int b = warp; b < cb1 - cb0; b += GT / 32) {
                double bf[KSMAX];
#pragma unroll
                for (int ks = 0; ks < KSMAX; ++ks) {
                    const int r = ks * 4 + (lane & 3), k = lane >> 2;
                    bf[ks] = (ks < KS && r < R && k < L) ? w2s[r * nz + b * L + k] : 0.0;
                }
                double* ps = psi + b * L3;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    double c[2] = {0.0, 0.0};
#pragma unroll
                    for (int ks = 0; ks < KSMAX; ++ks)
                        if (ks < KS) dmma884(c, af[mt][ks], bf[ks]);
                    const int row = mt * 8 + (lane >> 2), k0 = 2 * (lane & 3);
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc)
                        if (row < L2 && k0 + cc < L) {
                            ps[row * L + k0 + cc] = c[cc];
                            if (a.psi_cells)
                                a.psi_cells[(int64_t)(cell0 + b) * L3 + row * L + k0 + cc] = c[cc];
                        }
                }
            }
        } else {
            for (int e = tid; e < (cb1 - cb0) * L3; e += GT) {
                const int b = e / L3, node = e % L3;
                const int ij = node / L, k = node % L;
                const double* wr = w2s + b * L + k;
                double s = 0.0;
                for (int r = 0; r < R; ++r) s = fma(wr[r * nz], b2s[ij * R + r], s);
                psi[e] = s;
                if (a.psi_cells) a.psi_cells[(int64_t)(cell0 + b) * L3 + node] = s;
            }
        }
        __syncthreads();
        TRACE_MARK(1, 2);
        if (MONO && MODE != PSI_ONLY && !(GATHER_SKIP & 1) && cb1 - cb0 <= kGatherTab && !(GATHER_PAIRS && a.gpairs)) {
            // cell starts and z axes of the batch in shared memory; each thread
            // walks its particles in increasing order, so its cell only advances
            const int nb = cb1 - cb0;
            for (int e = tid; e <= nb; e += GT) gcst[e] = a.start[cell0 + e];
            for (int e = tid; e < nb; e += GT) gax[e] = a.cellax[2][cb0 + e];
            __syncthreads();
            const int s0 = gcst[0], s1 = gcst[nb];
            int cc = 0;
            double tmax = 0.0;
            RecStream rs{&a, s1, GT};
            rs.init(s0 + tid);
            for (int s = s0 + tid; s < s1; s += GT) {
                int dst;
                const double4 p = rs.next(s, dst);  // software prefetch of the next particle
                while (gcst[cc + 1] <= s) ++cc;
                const double* ps = psi + cc * L3;
                const double4 x2 = gax[cc];  // (lo, hi, mid, inv)
                double t[3];
                t[0] = (p.x - ax0.mid) * ax0.inv;
                t[1] = (p.y - ax1.mid) * ax1.inv;
                t[2] = (p.z - x2.z) * x2.w;
                tmax = fmax(tmax, fmax(fabs(t[0]), fmax(fabs(t[1]), fabs(t[2]))));
                double z = 0.0;
                if (GATHER_SKIP & 2) {
                    z = t[0] + t[1] + t[2] + ps[0];
                } else {
                    // ps = monomial coefficients C[a][b][c] of this cell's potential:
                    // z = sum_a t0^a sum_b t1^b sum_c t2^c C[a][b][c] (nested Horner)
#pragma unroll
                    for (int i = L - 1; i >= 0; --i) {
                        double zb = 0.0;
#pragma unroll
                        for (int j = L - 1; j >= 0; --j) {
                            const double* row = ps + (i * L + j) * L;
                            double zc = row[L - 1];
#pragma unroll
                            for (int k = L - 2; k >= 0; --k) zc = fma(zc, t[2], row[k]);
                            zb = fma(zb, t[1], zc);
                        }
                        z = fma(z, t[0], zb);
                    }
                }
                a.out[dst] = z - corr;
            }
            // tensor_weights' out-of-cell check, |t| <= 1 + 2e-12 (slack 1e-12 of the width)
            if (__ballot_sync(0xffffffffu, !(tmax <= 1.0 + 2e-12)) && (tid & 31) == 0)
                atomicOr(&a.bad[1], 1ull);
        } else if (MONO && MODE != PSI_ONLY && !(GATHER_SKIP & 1) && cb1 - cb0 <= kGatherTab) {
            // cell starts and z axes of the batch in shared memory; each thread
            // walks its particles in increasing order, so its cell only advances.
            // A thread takes two adjacent particles (s, s + 1): in the same cell
            // for the whole warp (the common case, warp vote) every coefficient
            // read from shared memory feeds both Horner chains, which halves the
            // shared-memory wavefronts that bound this loop.
            const int nb = cb1 - cb0;
            for (int e = tid; e <= nb; e += GT) gcst[e] = a.start[cell0 + e];
            for (int e = tid; e < nb; e += GT) gax[e] = a.cellax[2][cb0 + e];
            __syncthreads();
            const int s0 = gcst[0], s1 = gcst[nb];
            int cc = 0;
            double tmax = 0.0;
            int sb = s0 + 2 * tid;
            RecStream ra{&a, s1, 2 * GT}, rb{&a, s1, 2 * GT};
            ra.init(sb);
            rb.init(sb + 1);
            // nested Horner over the monomial coefficients C[a][b][c] of a cell:
            // z = sum_a t0^a sum_b t1^b sum_c t2^c C[a][b][c]
            auto horner1 = [&](const double* ps, const double (&t)[3]) {
                double z = 0.0;
#pragma unroll
                for (int i = L - 1; i >= 0; --i) {
                    double zb = 0.0;
#pragma unroll
                    for (int j = L - 1; j >= 0; --j) {
                        const double* row = ps + (i * L + j) * L;
                        double zc = row[L - 1];
#pragma unroll
                        for (int k = L - 2; k >= 0; --k) zc = fma(zc, t[2], row[k]);
                        zb = fma(zb, t[1], zc);
                    }
                    z = fma(z, t[0], zb);
                }
                return z;
            };
            // warp-uniform trip count (lane 0 holds the warp's lowest pair)
            for (int wb = s0 + 64 * (tid >> 5); wb < s1; wb += 2 * GT, sb += 2 * GT) {
                int d0, d1;
                const double4 p0 = ra.next(sb, d0), p1 = rb.next(sb + 1, d1);  // prefetched pair
                const bool has0 = sb < s1, has1 = sb + 1 < s1;
                while (gcst[cc + 1] <= min(sb, s1 - 1)) ++cc;
                int cc1 = cc;
                while (gcst[cc1 + 1] <= min(sb + 1, s1 - 1)) ++cc1;
                const double4 xa = gax[cc], xb = gax[cc1];  // (lo, hi, mid, inv)
                double ta[3], tb[3];
                ta[0] = (p0.x - ax0.mid) * ax0.inv;
                ta[1] = (p0.y - ax1.mid) * ax1.inv;
                ta[2] = (p0.z - xa.z) * xa.w;
                tb[0] = (p1.x - ax0.mid) * ax0.inv;
                tb[1] = (p1.y - ax1.mid) * ax1.inv;
                tb[2] = (p1.z - xb.z) * xb.w;
                if (has0) tmax = fmax(tmax, fmax(fabs(ta[0]), fmax(fabs(ta[1]), fabs(ta[2]))));
                if (has1) tmax = fmax(tmax, fmax(fabs(tb[0]), fmax(fabs(tb[1]), fabs(tb[2]))));
                double za, zb2;
                if (GATHER_SKIP & 2) {
                    za = ta[0] + ta[1] + ta[2] + psi[cc * L3];
                    zb2 = tb[0] + tb[1] + tb[2] + psi[cc1 * L3];
                } else if (__all_sync(0xffffffffu, cc1 == cc)) {
                    const double* ps = psi + cc * L3;
                    za = 0.0;
                    zb2 = 0.0;
#pragma unroll
                    for (int i = L - 1; i >= 0; --i) {
                        double ya = 0.0, yb = 0.0;
#pragma unroll
                        for (int j = L - 1; j >= 0; --j) {
                            const double* row = ps + (i * L + j) * L;
                            double xa_ = row[L - 1], xb_ = xa_;
#pragma unroll
                            for (int k = L - 2; k >= 0; --k) {
                                const double ck = row[k];
                                xa_ = fma(xa_, ta[2], ck);
                                xb_ = fma(xb_, tb[2], ck);
                            }
                            ya = fma(ya, ta[1], xa_);
                            yb = fma(yb, tb[1], xb_);
                        }
                        za = fma(za, ta[0], ya);
                        zb2 = fma(zb2, tb[0], yb);
                    }
                } else {
                    za = horner1(psi + cc * L3, ta);
                    zb2 = horner1(psi + cc1 * L3, tb);
                }
                if (has0) a.out[d0] = za - corr;
                if (has1) a.out[d1] = zb2 - corr;
            }
            // tensor_weights' out-of-cell check, |t| <= 1 + 2e-12 (slack 1e-12 of the width)
            if (__ballot_sync(0xffffffffu, !(tmax <= 1.0 + 2e-12)) && (tid & 31) == 0)
                atomicOr(&a.bad[1], 1ull);
        } else if (MODE != PSI_ONLY && !(GATHER_SKIP & 1)) {
            const int s0 = a.start[cell0], s1 = a.start[cell0 + (cb1 - cb0)];
            RecStream rs{&a, s1, GT};
            rs.init(s0 + tid);
            for (int s = s0 + tid; s < s1; s += GT) {
                int dst;
                const double4 p = rs.next(s, dst);  // software prefetch of the next particle
                const int c2 = axis_cell(p.z, g.center[2], g.radius, g.K[2], g.inv_diam);
                const double* ps = psi + (c2 - cb0) * L3;
                const CellAxis ax2 = cell_axis_tab(a.cellax[2], c2);
                double z = 0.0;
                if (GATHER_SKIP & 2) {
                    z = p.x + p.y + p.z + ps[0];
                } else if (MONO) {
                    // ps = monomial coefficients C[a][b][c] of this cell's potential:
                    // z = sum_a t0^a sum_b t1^b sum_c t2^c C[a][b][c] (nested Horner)
                    double t[3];
                    const CellAxis* axs[3] = {&ax0, &ax1, &ax2};
                    const double yv[3] = {p.x, p.y, p.z};
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const CellAxis& A = *axs[d];
                        const double slack = 1e-12 * (A.hi - A.lo);
                        if (yv[d] < A.lo - slack || yv[d] > A.hi + slack) atomicOr(&a.bad[1], 1ull);
                        t[d] = (yv[d] - A.mid) * A.inv;
                    }
#pragma unroll
                    for (int i = L - 1; i >= 0; --i) {
                        double zb = 0.0;
#pragma unroll
                        for (int j = L - 1; j >= 0; --j) {
                            const double* row = ps + (i * L + j) * L;
                            double zc = row[L - 1];
#pragma unroll
                            for (int k = L - 2; k >= 0; --k) zc = fma(zc, t[2], row[k]);
                            zb = fma(zb, t[1], zc);
                        }
                        z = fma(z, t[0], zb);
                    }
                } else {
                    double w0[L], w1[L], w2[L];
                    lagrange_fast<L>(lc, ax0.lo, ax0.hi, ax0.mid, ax0.inv, p.x, w0, a.bad);
                    lagrange_fast<L>(lc, ax1.lo, ax1.hi, ax1.mid, ax1.inv, p.y, w1, a.bad);
                    lagrange_fast<L>(lc, ax2.lo, ax2.hi, ax2.mid, ax2.inv, p.z, w2, a.bad);
                    // z = sum_k w2[k] sum_(i,j) (w0[i] w1[j]) psi[i][j][k]
                    double acc[L];
#pragma unroll
                    for (int k = 0; k < L; ++k) acc[k] = 0.0;
#pragma unroll
                    for (int i = 0; i < L; ++i)
#pragma unroll
                        for (int j = 0; j < L; ++j) {
                            const double tt = w0[i] * w1[j];
                            const double* row = ps + (i * L + j) * L;
#pragma unroll
                            for (int k = 0; k < L; ++k) acc[k] = fma(tt, row[k], acc[k]);
                        }
#pragma unroll
                    for (int k = 0; k < L; ++k) z = fma(w2[k], acc[k], z);
                }
                a.out[dst] = z - corr;
            }
        }
        __syncthreads();
        TRACE_MARK(1, 3);
    }
}

// ---- cell-chunk gather (the monomial hot path where cells hold >= 64 particles) ----
// The nested-Horner gather above is bound by shared-memory wavefronts: every
// lane reads all L^3 coefficients of its cell for each pair of particles, and a
// warp of adjacent pairs spans two cells most of the time (ncu, config 3: 6.6
// wavefronts per particle, data pipe 60% busy, FP64 pipe 32%). Here a warp takes
// an exact quarter of the batch's particles and walks them cell by cell in
// chunks of up to 128 from ONE cell: lane l evaluates particles l, l + 32,
// l + 64, l + 96 of the chunk as up to four interleaved Horner chains, so each
// coefficient is one broadcast read feeding up to 128 particles (about 2
// wavefronts per particle at 108 per cell) and the chains hide the DFMA
// latency. The records of the next chunk stream into a lane-private cp.async
// ring (x, y as one 16-byte copy, z as one 8-byte copy) while the current one
// is evaluated. Results, zero mode and the out-of-cell check are as above.
#ifndef GATHER_CC
#define GATHER_CC 1
#endif
constexpr int kCcChains = 4;
constexpr int kCcChunk = 32 * kCcChains;
constexpr int kCcStageDoubles = 4 * kCcChunk * 3;  // one ring stage: 4 warps x 128 x (x, y, z)
// Shared-memory layout (doubles): b2s | psi | ring stage 0 | scratch | w2s. The
// prologue scratch (G .* F, the x-expanded core, the W0 / W1 column rows) is
// dead once b2s exists, so ring stage 1 lies on top of it; stage 0 is separate:
// the first chunk's records are requested before the expansions run.
__host__ __device__ constexpr int gather_cc_scratch_doubles(int L, int R) {
    const int pro = R * R * R + L * R * R + 2 * R * L;
    return pro > kCcStageDoubles ? pro : kCcStageDoubles;
}
// offsets rounded to 16 bytes (cp.async and the 128-bit coefficient reads)
__host__ __device__ constexpr int gather_cc_psi_off(int L, int R) { return (L * L * R + 1) & ~1; }
__host__ __device__ constexpr int gather_cc_ring_off(int L, int R, int cb) {
    return gather_cc_psi_off(L, R) + ((cb * L * L * L + 1) & ~1);
}
__host__ __device__ constexpr int gather_cc_scr_off(int L, int R, int cb) {
    return gather_cc_ring_off(L, R, cb) + kCcStageDoubles;
}
__host__ __device__ constexpr size_t gather_cc_smem_doubles(int L, int R, int cb) {
    return (size_t)gather_cc_scr_off(L, R, cb) + (size_t)gather_cc_scratch_doubles(L, R) +
           (size_t)R * cb * L;
}

// z[u] = sum_abc C[a][b][c] t0[u]^a t1[u]^b t2[u]^c for NCH particles of one cell
// (nested Horner; the a loop is kept rolled: the body is already 36 NCH DFMAs)
template <int L, int NCH>
__device__ __forceinline__ void horner_chains(const double* __restrict__ ps, const double (&t0)[NCH],
                                              const double (&t1)[NCH], const double (&t2)[NCH],
                                              double (&z)[NCH]) {
#pragma unroll
    for (int u = 0; u < NCH; ++u) z[u] = 0.0;
#pragma unroll 1
    for (int i = L - 1; i >= 0; --i) {
        double zb[NCH];
        const double* rowi = ps + i * L * L;
#pragma unroll
        for (int j = L - 1; j >= 0; --j) {
            const double* row = rowi + j * L;
            double c[L];
            if (L % 2 == 0) {
#pragma unroll
                for (int k = 0; k < L; k += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(row + k);
                    c[k] = v.x;
                    c[k + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int k = 0; k < L; ++k) c[k] = row[k];
            }
            double zc[NCH];
#pragma unroll
            for (int u = 0; u < NCH; ++u) zc[u] = c[L - 1];
#pragma unroll
            for (int k = L - 2; k >= 0; --k)
#pragma unroll
                for (int u = 0; u < NCH; ++u) zc[u] = fma(zc[u], t2[u], c[k]);
#pragma unroll
            for (int u = 0; u < NCH; ++u) zb[u] = j == L - 1 ? zc[u] : fma(zb[u], t1[u], zc[u]);
        }
#pragma unroll
        for (int u = 0; u < NCH; ++u) z[u] = fma(z[u], t0[u], zb[u]);
    }
}

// One chunk: particles cbase + lane + 32 u (u < NCH) of the cell whose
// coefficients are at ps; records from the lane's ring slots.
template <int L, int NCH>
__device__ __forceinline__ void gather_cc_chunk(const ColumnArgs& a, const double* __restrict__ ps,
                                                const double2* __restrict__ rxy,
                                                const double* __restrict__ rz, int cbase, int end,
                                                int lane, const CellAxis& ax0, const CellAxis& ax1,
                                                const double4& x2, double corr, double& tmax,
                                                long long* hacc = nullptr) {
    double t0[NCH], t1[NCH], t2[NCH], z[NCH];
    int dst[NCH];
#pragma unroll
    for (int u = 0; u < NCH; ++u) {
        const int s = cbase + lane + 32 * u;
        const bool ok = s < end;
        dst[u] = ok ? __ldg(a.perm + s) : -1;
        const double2 xy = rxy[lane + 32 * u];
        const double zz = rz[lane + 32 * u];
        t0[u] = ok ? (xy.x - ax0.mid) * ax0.inv : 0.0;
        t1[u] = ok ? (xy.y - ax1.mid) * ax1.inv : 0.0;
        t2[u] = ok ? (zz - x2.z) * x2.w : 0.0;
        tmax = fmax(tmax, fmax(fabs(t0[u]), fmax(fabs(t1[u]), fabs(t2[u]))));
    }
    TRACE_CLK(h0);
    horner_chains<L, NCH>(ps, t0, t1, t2, z);
    TRACE_CLK(h1);
#ifdef KB_TRACE
    if (hacc) *hacc += h1 - h0;
#endif
#pragma unroll
    for (int u = 0; u < NCH; ++u)
        if (dst[u] >= 0) a.out[dst[u]] = z[u] - corr;
}

template <int L, int MINB, int RC>
__global__ void __launch_bounds__(128, MINB) k_gather_cc(ColumnArgs a, int cells_per_batch) {
    constexpr int L2 = L * L, L3 = L2 * L, NW = 4, NTH = 128;
    const Geometry& g = a.g;
    const int R = RC ? RC : g.R;  // RC: compile-time R (unrolled expansions), 0 = any R <= 16
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const ColumnRange cr = column_range(g, a.S);
    extern __shared__ double sm[];
    double* b2s = sm;                                         // [L^2][R]
    double* psi = sm + gather_cc_psi_off(L, R);               // [cells_per_batch][L^3]
    double* ring0 = sm + gather_cc_ring_off(L, R, cells_per_batch);
    double* scr = sm + gather_cc_scr_off(L, R, cells_per_batch);  // prologue scratch, then ring stage 1
    double* w2s = scr + gather_cc_scratch_doubles(L, R);      // [R][cells_per_batch * L]
    __shared__ int gcst[kGatherTab + 1];
    __shared__ double4 gax[kGatherTab];
    TRACE_MARK(1, 0);
    const int RR = R * R, R3 = RR * R;
    double* h = scr;           // [R^3]  G .* F
    double* v = h + R3;        // [L][R][R]
    double* w01 = v + L * RR;  // [2][R][L]
    // ring stage st of this warp: (x, y) pairs then z
    auto stage_xy = [&](int st) { return reinterpret_cast<double2*>(st ? scr : ring0) + warp * kCcChunk; };
    auto stage_z = [&](int st) { return (st ? scr : ring0) + NW * kCcChunk * 2 + warp * kCcChunk; };
    const CellAxis ax0 = cell_axis_tab(a.cellax[0], cr.c0), ax1 = cell_axis_tab(a.cellax[1], cr.c1);
    const bool fused = a.B2 == nullptr;
    double corr = 0.0;  // fused: the zero mode carries the correction; else read after pdl_wait()
    double tmax = 0.0;
    for (int cb0 = cr.zb; cb0 < cr.ze; cb0 += cells_per_batch) {
        const bool first = cb0 == cr.zb;
        const int cb1 = min(cr.ze, cb0 + cells_per_batch), nb = cb1 - cb0;
        const int cell0 = (cr.c0 * g.K[1] + cr.c1) * g.K[2] + cb0;
        const int nz = nb * L;
        {
            // every global load of the batch's tables (and, in the first batch,
            // of the column's core and W rows) is in flight before the first use
            constexpr int WU = 16, HU = 6;  // R <= 16 rows of the W2 slice, one z column per thread
            double wv[WU], gv[HU], fv[HU], wa = 0.0, wb = 0.0;
            const bool w2_regs = nz <= NTH, h_regs = R3 <= NTH * HU;
            if (w2_regs && tid < nz) {
                const double* wsrc = a.W2 + cb0 * L + tid;
#pragma unroll
                for (int u = 0; u < WU; ++u)
                    if (u < R) wv[u] = __ldg(wsrc + (int64_t)u * g.n[2]);
            }
            // The cell starts come from the sort, an earlier kernel of the launch
            // chain: every kernel of the chain triggers its dependent when it
            // starts, so before pdl_wait() only plan constants may be read.
            int st0 = (!first && tid <= nb) ? __ldg(a.start + cell0 + tid) : 0;
            double4 axv = make_double4(0.0, 0.0, 0.0, 0.0);
            if (tid < nb) axv = a.cellax[2][cb0 + tid];
            if (first && fused) {
                if (h_regs) {
#pragma unroll
                    for (int u = 0; u < HU; ++u)
                        if (tid + NTH * u < R3) gv[u] = __ldg(a.Gc + tid + NTH * u);
                }
                if (tid < R * L) {
                    wa = a.W0[(int64_t)(tid / L) * g.n[0] + cr.c0 * L + tid % L];
                    wb = a.W1[(int64_t)(tid / L) * g.n[1] + cr.c1 * L + tid % L];
                }
            }
            if (tid < nb) gax[tid] = axv;
            if (w2_regs) {
                if (tid < nz) {
#pragma unroll
                    for (int u = 0; u < WU; ++u)
                        if (u < R) w2s[u * nz + tid] = wv[u];
                }
            } else {
                for (int e = tid; e < R * nz; e += NTH)
                    w2s[e] = __ldg(a.W2 + (int64_t)(e / nz) * g.n[2] + cb0 * L + e % nz);
            }
            if (first && fused) {
                // Everything above is independent of the summed core: under a
                // programmatic dependent launch it ran while the core sum did.
                pdl_wait();
                if (tid <= nb) st0 = __ldg(a.start + cell0 + tid);
                double fq = 0.0;  // sum q (the last core entry), for the zero mode
                if (tid == 0) fq = __ldcg(a.Fc + R3);
                // zero mode, exactly: h[0] = (G[0] - c) sum q
                if (h_regs) {
#pragma unroll
                    for (int u = 0; u < HU; ++u)
                        if (tid + NTH * u < R3) fv[u] = __ldcg(a.Fc + tid + NTH * u);
#pragma unroll
                    for (int u = 0; u < HU; ++u)
                        if (tid + NTH * u < R3)
                            h[tid + NTH * u] = (u == 0 && tid == 0) ? (gv[0] - a.correction) * fq : gv[u] * fv[u];
                } else {
                    for (int e = tid; e < R3; e += NTH)
                        h[e] = e == 0 ? (__ldg(a.Gc) - a.correction) * fq : __ldg(a.Gc + e) * __ldcg(a.Fc + e);
                }
                if (tid < R * L) {
                    w01[tid] = wa;
                    w01[R * L + tid] = wb;
                }
                for (int e = NTH + tid; e < R * L; e += NTH) {  // R * L > 128 only for R > 16
                    w01[e] = a.W0[(int64_t)(e / L) * g.n[0] + cr.c0 * L + e % L];
                    w01[R * L + e] = a.W1[(int64_t)(e / L) * g.n[1] + cr.c1 * L + e % L];
                }
            } else if (first) {
                pdl_wait();
                if (tid <= nb) st0 = __ldg(a.start + cell0 + tid);
                corr = a.corr ? *a.corr : 0.0;
                for (int e = tid; e < L2 * R; e += NTH) {
                    const int ij = e / R, r = e % R, i = ij / L, j = ij % L;
                    b2s[e] = a.B2[((int64_t)(cr.c0 * L + i) * g.n[1] + cr.c1 * L + j) * R + r];
                }
            }
            if (tid <= nb) gcst[tid] = st0;
        }
        __syncthreads();
        if (first) TRACE_MARK(1, 7);
        // The warp's particle range of this batch and its first chunk's records:
        // requested now, they arrive while the expansions below run. (The cell
        // starts are read with explicit shared loads: through the lambdas below
        // the table would be read with generic loads and a window-address rebuild.)
        const unsigned gcst_sa = (unsigned)__cvta_generic_to_shared(gcst);
        auto gc = [=](int e) {
            int v;
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(gcst_sa + 4u * (unsigned)e));
            return v;
        };
        const int P0 = gc(0), P1 = gc(nb);
        const int pw0 = P0 + (int)((long long)(P1 - P0) * warp / NW);
        const int pw1 = P0 + (int)((long long)(P1 - P0) * (warp + 1) / NW);
        int cc = 0, pc = 0, pbase = pw0, cbase = pw0, pslot = 0, cslot = 0;
        int pend = pw0, cend = pw0;  // ends (within the warp's range) of the producer's / consumer's cell
        if (pw0 < pw1) {
            while (gc(cc + 1) <= pw0) ++cc;
            pc = cc;
            pend = cend = min(gc(cc + 1), pw1);
        }
        auto issue = [&]() {
            if (pbase < pw1) {
                const int end = min(pbase + kCcChunk, pend);
                double2* dxy = stage_xy(pslot);
                double* dz = stage_z(pslot);
#pragma unroll
                for (int u = 0; u < kCcChains; ++u) {
                    const int s = pbase + lane + 32 * u;
                    if (s < end) {
                        const char* src = reinterpret_cast<const char*>(a.sp + s);
                        cp_async16_sm(dxy + lane + 32 * u, src);
                        cp_async8_sm(dz + lane + 32 * u, src + 16);
                    }
                }
                pbase = end;
                if (pbase >= pend && pbase < pw1) {  // next non-empty cell
                    int e;
                    do {
                        ++pc;
                        e = gc(pc + 1);
                    } while (pbase >= e);
                    pend = min(e, pw1);
                }
            }
            cp_async_commit();
            pslot ^= 1;
        };
        issue();  // stage 0 (never aliased)
        if (first && fused) {
            // fused backward y, x expansions (the U_0, U_1 phases of spkmv) for this column
            if constexpr (RC > 0) {
                // every thread's outputs at once: the loads of all of them are in flight together
                constexpr int NV = L * RC * RC, IT = (NV + NTH - 1) / NTH;
                double sv[IT];
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                    const int e = min(tid + it * NTH, NV - 1);
                    const int i = e / (RC * RC), rr = e % (RC * RC);
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int r0 = 0; r0 < RC; r0 += 2) {
                        s0 = fma(w01[r0 * L + i], h[r0 * RC * RC + rr], s0);
                        if (r0 + 1 < RC) s1 = fma(w01[(r0 + 1) * L + i], h[(r0 + 1) * RC * RC + rr], s1);
                    }
                    sv[it] = s0 + s1;
                }
#pragma unroll
                for (int it = 0; it < IT; ++it)
                    if (tid + it * NTH < NV) v[tid + it * NTH] = sv[it];
            } else {
                for (int e = tid; e < L * RR; e += NTH) {
                    const int i = e / RR, rr = e % RR;
                    double s = 0.0;
                    for (int r0 = 0; r0 < R; ++r0) s = fma(w01[r0 * L + i], h[r0 * RR + rr], s);
                    v[e] = s;
                }
            }
            __syncthreads();
            if constexpr (RC > 0) {
                constexpr int NB = L2 * RC, IT = (NB + NTH - 1) / NTH;
                double sv[IT];
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                    const int e = min(tid + it * NTH, NB - 1);
                    const int ij = e / RC, r2 = e % RC, i = ij / L, j = ij % L;
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int r1 = 0; r1 < RC; r1 += 2) {
                        s0 = fma(w01[RC * L + r1 * L + j], v[i * RC * RC + r1 * RC + r2], s0);
                        if (r1 + 1 < RC)
                            s1 = fma(w01[RC * L + (r1 + 1) * L + j], v[i * RC * RC + (r1 + 1) * RC + r2], s1);
                    }
                    sv[it] = s0 + s1;
                }
#pragma unroll
                for (int it = 0; it < IT; ++it)
                    if (tid + it * NTH < NB) b2s[tid + it * NTH] = sv[it];
            } else {
                for (int e = tid; e < L2 * R; e += NTH) {
                    const int ij = e / R, r2 = e % R, i = ij / L, j = ij % L;
                    double s = 0.0;
                    for (int r1 = 0; r1 < R; ++r1) s = fma(w01[R * L + r1 * L + j], v[i * RR + r1 * R + r2], s);
                    b2s[e] = s;
                }
            }
        }
        if (first) {
            __syncthreads();
            TRACE_MARK(1, 1);
        }
        {
            // psi_cell[(i,j)][k] = sum_r B2col[(i,j)][r] W2[r][c2 L + k] on DMMA (R <= 16).
            // Row r = 0 of the monomial W2 is exactly (1, 0, ..., 0) in every cell
            // (k_factor_wl), so it adds B2col[(i,j)][0] at k = 0 and the product
            // runs over r = 1 .. R-1 (R = 9: two k-steps, no padding).
            constexpr int MT = (L2 + 7) / 8, KSMAX = RC ? (RC + 2) / 4 : 4;
            const int R1 = R - 1, KS = (R1 + 3) / 4;
            double af[MT][KSMAX], b0[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int row = mt * 8 + (lane >> 2);
                b0[mt] = ((lane & 3) == 0 && row < L2) ? b2s[row * R] : 0.0;
#pragma unroll
                for (int ks = 0; ks < KSMAX; ++ks) {
                    const int r = ks * 4 + (lane & 3);
                    af[mt][ks] = (ks < KS && row < L2 && r < R1) ? b2s[row * R + 1 + r] : 0.0;
                }
            }
            for (int b = warp; b < nb; b += NW) {
                double bf[KSMAX];
#pragma unroll
                for (int ks = 0; ks < KSMAX; ++ks) {
                    const int r = ks * 4 + (lane & 3), k = lane >> 2;
                    bf[ks] = (ks < KS && r < R1 && k < L) ? w2s[(1 + r) * nz + b * L + k] : 0.0;
                }
                double* ps = psi + b * L3;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    double c[2] = {b0[mt], 0.0};
#pragma unroll
                    for (int ks = 0; ks < KSMAX; ++ks)
                        if (ks < KS) dmma884(c, af[mt][ks], bf[ks]);
                    const int row = mt * 8 + (lane >> 2), k0 = 2 * (lane & 3);
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
                        if (row < L2 && k0 + q2 < L) {
                            ps[row * L + k0 + q2] = c[q2];
                            if (a.psi_cells)
                                a.psi_cells[(int64_t)(cell0 + b) * L3 + row * L + k0 + q2] = c[q2];
                        }
                }
            }
        }
        __syncthreads();  // psi complete; the scratch is free for ring stage 1
        TRACE_MARK(1, 2);
        if (pw0 < pw1) {
            TRACE_DECL(tr_wait);
            TRACE_DECL(tr_work);
            TRACE_DECL(tr_chunks);
            TRACE_DECL(tr_horner);
            while (cbase < pw1) {
                const int end = min(cbase + kCcChunk, cend);
                TRACE_CLK(tr0);
                issue();
                cp_async_wait<1>();
                TRACE_CLK(tr1);
                const double* ps = psi + cc * L3;
                const double4 x2 = gax[cc];  // (lo, hi, mid, inv)
                const double2* cxy = stage_xy(cslot);
                const double* cz = stage_z(cslot);
                switch ((end - cbase + 31) >> 5) {
                    case 1: gather_cc_chunk<L, 1>(a, ps, cxy, cz, cbase, end, lane, ax0, ax1, x2, corr, tmax, TRACE_PTR(tr_horner)); break;
                    case 2: gather_cc_chunk<L, 2>(a, ps, cxy, cz, cbase, end, lane, ax0, ax1, x2, corr, tmax, TRACE_PTR(tr_horner)); break;
                    case 3: gather_cc_chunk<L, 3>(a, ps, cxy, cz, cbase, end, lane, ax0, ax1, x2, corr, tmax, TRACE_PTR(tr_horner)); break;
                    default: gather_cc_chunk<L, 4>(a, ps, cxy, cz, cbase, end, lane, ax0, ax1, x2, corr, tmax, TRACE_PTR(tr_horner));
                }
                TRACE_CLK(tr2);
                TRACE_ACC(tr_wait, tr0, tr1);
                TRACE_ACC(tr_work, tr1, tr2);
                TRACE_ACC(tr_chunks, 0, (end - cbase + 31) >> 5);
                cslot ^= 1;
                cbase = end;
                if (cbase >= cend && cbase < pw1) {
                    int e;
                    do {
                        ++cc;
                        e = gc(cc + 1);
                    } while (cbase >= e);
                    cend = min(e, pw1);
                }
            }
            TRACE_PUT(1, 4, tr_wait);
            TRACE_PUT(1, 5, tr_work);
            TRACE_PUT(1, 6, tr_chunks);
            TRACE_PUT(1, 8, tr_horner);
        }
        cp_async_wait<0>();
        __syncthreads();
        TRACE_MARK(1, 3);
    }
    // tensor_weights' out-of-cell check, |t| <= 1 + 2e-12 (slack 1e-12 of the width)
    if (__ballot_sync(0xffffffffu, !(tmax <= 1.0 + 2e-12)) && lane == 0) atomicOr(&a.bad[1], 1ull);
}

size_t spread_smem(const Geometry& g) {
    const int L = g.L;
    return sizeof(double) * ((size_t)L * L * L + (size_t)L * L * g.R + (size_t)g.R * L +
                             (size_t)kChunk * 3 * L);
}

#ifndef GATHER_BATCH_KB
#define GATHER_BATCH_KB 28  // shared memory for the batch's cell coefficients
#endif
// Cells per gather batch: 28 KB of coefficients in equal batches, or the
// whole column segment when it fits in 40 KB and the column CTAs make one
// wave at three per SM (each batch costs a serial load -> expand -> evaluate
// round; config 3: one batch of 21 cells, 47.8 -> 46.4 us). Grids of many
// columns keep the smaller batch: their fourth CTA per SM is worth more
// (config 4: 3 rounds of 15/14/14 cells, 185 us; 40 KB batches 204 us;
// 24 KB, 4 rounds, 192 us).
int gather_batch(const Geometry& g, int S = 1) {
    const int L3 = g.L * g.L * g.L;
    const int seg = (g.z_hi - g.z_lo + S - 1) / std::max(1, S);
    if (block_columns(g) * S <= 3 * sm_count() && seg <= kGatherTab && (size_t)seg * L3 * sizeof(double) <= 40 * 1024)
        return std::max(1, seg);
    const int cap = std::max(1, (GATHER_BATCH_KB * 1024) / (int)(sizeof(double) * L3));
    // equal batches for the same number of rounds: no short tail round
    // (config 4: 43 cells as 11 + 11 + 11 + 10, not 14 + 14 + 14 + 1)
    const int rounds = (std::max(1, seg) + cap - 1) / cap;
    return (std::max(1, seg) + rounds - 1) / rounds;
}


template <int L, bool MONO>
void launch_spread_mma_t(const ColumnArgs& a, bool want_fwd, cudaStream_t s) {
    const int R = a.g.R;
    const bool fits = spread_epilogue_doubles(L, R) <= SpreadTile<L>::stage;
    const size_t smem = sizeof(double) * (SpreadTile<L>::NW * spread_warp_doubles<L>(R) +
                                          (fits ? 0 : (size_t)spread_epilogue_doubles(L, R)));
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_spread_mma<L, MONO>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    if (smem > 200 * 1024) throw Error(KPME_GPU_INVALID_ARGUMENT, "spread: tile too large");
    const int grid = block_columns(a.g) * a.S;
    k_spread_mma<L, MONO><<<grid, 128, smem, s>>>(a, want_fwd ? 1 : 0);
    KB_CHECK_LAUNCH();
}

#ifndef SPREAD_UV
#define SPREAD_UV 1
#endif
#ifndef SPREAD_F8
#define SPREAD_F8 1  // split-exponent spread for L = 4, 6
#endif
#ifndef DIRECT_RECORDS
#define DIRECT_RECORDS 1
#endif
template <int L>
bool launch_spread_f8_t(const ColumnArgs& a, bool want_fwd, cudaStream_t s) {
    if constexpr (L == 4 || L == 6) {
        const size_t smem = sizeof(double) * spread_f8_smem_doubles<L>(a.g.R, a.g.n[2]);
        if (!SPREAD_F8 || smem > 200 * 1024 || a.g.R > 32) return false;
        static PerDevice attr_once;
        once_per_device(attr_once, [&] {
            KB_CUDA(cudaFuncSetAttribute(k_spread_f8<L, 1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024));
            KB_CUDA(cudaFuncSetAttribute(k_spread_f8<L, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024));
            KB_CUDA(cudaFuncSetAttribute(k_spread_f8<L, 2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024));
            KB_CUDA(cudaFuncSetAttribute(k_spread_f8<L, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024));
            KB_CUDA(cudaFuncSetAttribute(k_spread_f8<L, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024));
        });
        const int grid = block_columns(a.g) * a.S;
        const bool waves = grid > 2 * 3 * sm_count() && smem * 4 <= 220 * 1024;
        // n-tiles of the W2 contraction over r = 1 .. R-1
        if (a.g.R <= 9 && waves)
            launch_pdl_if((pdl_mask() & 2) != 0, k_spread_f8<L, 1, 4>, dim3(grid), dim3(32 * F8_NW), smem, s, a, want_fwd ? 1 : 0);
        else if (a.g.R <= 9)
            launch_pdl_if((pdl_mask() & 2) != 0, k_spread_f8<L, 1, 3>, dim3(grid), dim3(32 * F8_NW), smem, s, a, want_fwd ? 1 : 0);
        else if (a.g.R <= 17 && waves)
            launch_pdl_if((pdl_mask() & 2) != 0, k_spread_f8<L, 2, 4>, dim3(grid), dim3(32 * F8_NW), smem, s, a, want_fwd ? 1 : 0);
        else if (a.g.R <= 17)
            launch_pdl_if((pdl_mask() & 2) != 0, k_spread_f8<L, 2, 3>, dim3(grid), dim3(32 * F8_NW), smem, s, a, want_fwd ? 1 : 0);
        else
            launch_pdl_if((pdl_mask() & 2) != 0, k_spread_f8<L, 4, 3>, dim3(grid), dim3(32 * F8_NW), smem, s, a, want_fwd ? 1 : 0);
        KB_CHECK_LAUNCH();
        return true;
    } else {
        return false;
    }
}

template <int L>
void launch_spread_uv_t(const ColumnArgs& a, bool want_fwd, cudaStream_t s) {
    if (launch_spread_f8_t<L>(a, want_fwd, s)) return;
    const size_t smem = sizeof(double) * spread_uv_smem_doubles<L>(a.g.R, a.g.n[2]);
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_spread_uv<L, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_spread_uv<L, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
    });
    if (smem > 200 * 1024) {  // very long columns: the staged-product kernel
        launch_spread_mma_t<L, true>(a, want_fwd, s);
        return;
    }
    const int grid = block_columns(a.g) * a.S;
    if (UV_SKIP & 8) {
        static double* scratch = nullptr;
        if (!scratch) {
            KB_CUDA(cudaMalloc(&scratch, sizeof(double) * 64 * 8 * (size_t)a.g.ncell));
            KB_CUDA(cudaMemcpyToSymbol(uv_scratch, &scratch, sizeof(scratch)));
        }
    }
    if (a.g.R <= 16)
        k_spread_uv<L, 2><<<grid, 32 * UV_NW, smem, s>>>(a, want_fwd ? 1 : 0);
    else
        k_spread_uv<L, 4><<<grid, 32 * UV_NW, smem, s>>>(a, want_fwd ? 1 : 0);
    KB_CHECK_LAUNCH();
}

template <int L>
void launch_spread_mma(const ColumnArgs& a, bool want_fwd, cudaStream_t s) {
    if (a.mono && SPREAD_UV)
        launch_spread_uv_t<L>(a, want_fwd, s);
    else if (a.mono)
        launch_spread_mma_t<L, true>(a, want_fwd, s);
    else
        launch_spread_mma_t<L, false>(a, want_fwd, s);
}

template <int L, int MODE, bool MONO>
void launch_gather_mode(const ColumnArgs& a, int grid, int cb, size_t smem, cudaStream_t s) {
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather_t<L, MODE, MONO>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    k_bwd_gather_t<L, MODE, MONO><<<grid, GT, smem, s>>>(a, cb);
}

template <int L>
void launch_gather_t(const ColumnArgs& a0, int mode, cudaStream_t s) {
    ColumnArgs a = a0;
#ifdef GATHER_S
    if (mode == GATHER_FROM_B2 && a.B2 == nullptr) a.S = std::max(1, std::min(GATHER_S, a.g.z_hi - a.g.z_lo));
#endif
    const int grid = block_columns(a.g) * a.S;
#ifdef GATHER_CB
    const int cb = std::min(gather_batch(a.g, a.S), GATHER_CB);
#else
    const int cb = gather_batch(a.g, a.S);
#endif
    const int R = a.g.R;
    const size_t smem = sizeof(double) * ((size_t)L * L * R + (size_t)cb * L * L * L +
                                          (size_t)R * R * R + (size_t)L * R * R +
                                          2 * (size_t)R * L + (size_t)R * cb * L);
    if constexpr (L == 4 || L == 6 || L == 8) {
        // cell-chunk gather: the monomial hot path where cells are full enough
        // (the plan's gpairs flag: >= 64 particles per cell on average)
        static const int cc_env = [] {
            const char* e = getenv("KPME_GATHER_CC");
            return e ? atoi(e) : -1;
        }();
        const bool cc_on = cc_env >= 0 ? cc_env != 0 : a.gpairs != 0;
        if (GATHER_CC && cc_on && mode == GATHER_FROM_B2 && a.mono && R <= 16 && !a.direct) {
            const int ccb = std::min(cb, kGatherTab);
            const size_t csm = sizeof(double) * gather_cc_smem_doubles(L, R, ccb);
            if (csm <= 200 * 1024) {
                static PerDevice cc_once;
                once_per_device(cc_once, [&] {
                    KB_CUDA(cudaFuncSetAttribute(k_gather_cc<L, 3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 200 * 1024));
                    KB_CUDA(cudaFuncSetAttribute(k_gather_cc<L, 4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 200 * 1024));
                    KB_CUDA(cudaFuncSetAttribute(k_gather_cc<L, 3, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 200 * 1024));
                    KB_CUDA(cudaFuncSetAttribute(k_gather_cc<L, 4, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 200 * 1024));
                });
                const bool waves = grid > 2 * 3 * sm_count() && csm * 4 <= 220 * 1024;
                if (R == 9 && waves)
                    launch_pdl_if((pdl_mask() & 8) != 0, k_gather_cc<L, 4, 9>, dim3(grid), dim3(128), csm, s, a, ccb);
                else if (R == 9)
                    launch_pdl_if((pdl_mask() & 8) != 0, k_gather_cc<L, 3, 9>, dim3(grid), dim3(128), csm, s, a, ccb);
                else if (waves)
                    launch_pdl_if((pdl_mask() & 8) != 0, k_gather_cc<L, 4, 0>, dim3(grid), dim3(128), csm, s, a, ccb);
                else
                    launch_pdl_if((pdl_mask() & 8) != 0, k_gather_cc<L, 3, 0>, dim3(grid), dim3(128), csm, s, a, ccb);
                KB_CHECK_LAUNCH();
                return;
            }
        }
    }
    switch (mode) {
        case GATHER_FROM_B2:
            if (a.mono && L <= 8)
                launch_gather_mode<L, GATHER_FROM_B2, true>(a, grid, cb, smem, s);
            else
                launch_gather_mode<L, GATHER_FROM_B2, false>(a, grid, cb, smem, s);
            break;
        case GATHER_FROM_CELLS:
            launch_gather_mode<L, GATHER_FROM_CELLS, false>(a, grid, cb, smem, s);
            break;
        default:
            launch_gather_mode<L, PSI_ONLY, false>(a, grid, cb, smem, s);
    }
    KB_CHECK_LAUNCH();
}

}  // namespace

bool direct_records_ok(const Geometry& g) {
    if (!DIRECT_RECORDS || !SPREAD_F8 || g.R > 32) return false;
    size_t smem;
    if (g.L == 4)
        smem = sizeof(double) * spread_f8_smem_doubles<4>(g.R, g.n[2]);
    else if (g.L == 6)
        smem = sizeof(double) * spread_f8_smem_doubles<6>(g.R, g.n[2]);
    else
        return false;
    return smem <= 200 * 1024;
}

void launch_spread_fwd(const ColumnArgs& a, int mode, bool want_fwd, cudaStream_t s) {
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_spread_fwd<SPREAD_PARTICLES>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_spread_fwd<SPREAD_FROM_CELLS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    if (mode == SPREAD_PARTICLES && a.g.L <= 8) {
        switch (a.g.L) {
            case 2: return launch_spread_mma<2>(a, want_fwd, s);
            case 3: return launch_spread_mma<3>(a, want_fwd, s);
            case 4: return launch_spread_mma<4>(a, want_fwd, s);
            case 5: return launch_spread_mma<5>(a, want_fwd, s);
            case 6: return launch_spread_mma<6>(a, want_fwd, s);
            case 7: return launch_spread_mma<7>(a, want_fwd, s);
            default: return launch_spread_mma<8>(a, want_fwd, s);
        }
    }
    const int grid = block_columns(a.g) * a.S;
    const size_t smem = spread_smem(a.g);
    if (mode == SPREAD_PARTICLES)
        k_spread_fwd<SPREAD_PARTICLES><<<grid, kThreads, smem, s>>>(a, want_fwd ? 1 : 0);
    else
        k_spread_fwd<SPREAD_FROM_CELLS><<<grid, kThreads, smem, s>>>(a, want_fwd ? 1 : 0);
    KB_CHECK_LAUNCH();
}

void launch_bwd_gather(const ColumnArgs& a, int mode, cudaStream_t s) {
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather<GATHER_FROM_B2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather<GATHER_FROM_CELLS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather<PSI_ONLY>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    switch (a.g.L) {
        case 2: return launch_gather_t<2>(a, mode, s);
        case 3: return launch_gather_t<3>(a, mode, s);
        case 4: return launch_gather_t<4>(a, mode, s);
        case 5: return launch_gather_t<5>(a, mode, s);
        case 6: return launch_gather_t<6>(a, mode, s);
        case 7: return launch_gather_t<7>(a, mode, s);
        case 8: return launch_gather_t<8>(a, mode, s);
        case 10: return launch_gather_t<10>(a, mode, s);
        case 12: return launch_gather_t<12>(a, mode, s);
        default: break;
    }
    const int grid = block_columns(a.g) * a.S;
    const int cb = gather_batch(a.g);
    const size_t smem =
        sizeof(double) * ((size_t)a.g.L * a.g.L * a.g.R + (size_t)cb * a.g.L * a.g.L * a.g.L);
    switch (mode) {
        case GATHER_FROM_B2:
            k_bwd_gather<GATHER_FROM_B2><<<grid, kThreads, smem, s>>>(a, cb);
            break;
        case GATHER_FROM_CELLS:
            k_bwd_gather<GATHER_FROM_CELLS><<<grid, kThreads, smem, s>>>(a, cb);
            break;
        default:
            k_bwd_gather<PSI_ONLY><<<grid, kThreads, smem, s>>>(a, cb);
    }
    KB_CHECK_LAUNCH();
}

}  // namespace kb

TRACE_READER(interp)
