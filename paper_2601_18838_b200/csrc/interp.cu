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

// Same exact key arithmetic as sort.cu (geometry.hpp:141-148).
__device__ __forceinline__ int axis_cell(double p, double c, double r, int K) {
    const double t = __ddiv_rn(__dmul_rn(__dsub_rn(p, __dsub_rn(c, r)), (double)K),
                               __dmul_rn(2.0, r));
    int idx = (int)floor(t);
    if (t == (double)idx && idx > 0) --idx;
    return idx < 0 ? 0 : (idx > K - 1 ? K - 1 : idx);
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
    r.col = blockIdx.x / S;
    r.seg = blockIdx.x % S;
    r.c0 = r.col / g.K[1];
    r.c1 = r.col % g.K[1];
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
                const int c2 = axis_cell(p.z, g.center[2], g.radius, g.K[2]);
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

size_t spread_smem(const Geometry& g) {
    const int L = g.L;
    return sizeof(double) * ((size_t)L * L * L + (size_t)L * L * g.R + (size_t)g.R * L +
                             (size_t)kChunk * 3 * L);
}

int gather_batch(const Geometry& g) {
    const int L3 = g.L * g.L * g.L;
    const int cap = (96 * 1024) / (int)(sizeof(double) * L3);
    return cap < 1 ? 1 : cap;
}

}  // namespace

void launch_spread_fwd(const ColumnArgs& a, int mode, bool want_fwd, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        KB_CUDA(cudaFuncSetAttribute(k_spread_fwd<SPREAD_PARTICLES>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_spread_fwd<SPREAD_FROM_CELLS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    const int grid = a.g.K[0] * a.g.K[1] * a.S;
    const size_t smem = spread_smem(a.g);
    if (mode == SPREAD_PARTICLES)
        k_spread_fwd<SPREAD_PARTICLES><<<grid, kThreads, smem, s>>>(a, want_fwd ? 1 : 0);
    else
        k_spread_fwd<SPREAD_FROM_CELLS><<<grid, kThreads, smem, s>>>(a, want_fwd ? 1 : 0);
    KB_CHECK_LAUNCH();
}

void launch_bwd_gather(const ColumnArgs& a, int mode, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather<GATHER_FROM_B2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather<GATHER_FROM_CELLS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_bwd_gather<PSI_ONLY>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    const int grid = a.g.K[0] * a.g.K[1] * a.S;
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
