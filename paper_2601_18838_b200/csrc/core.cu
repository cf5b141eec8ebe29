// core.cu -- SKP factor tables and the term-collapsed grid operator core.
//
// The reference applies, per SKP term lambda and axis a, the per-cell factor
// pair U = W(x)^T, V = diag(cbrt(w) * even_profile) W(x) (build_uv,
// symfourier.hpp:108-124; factor loop parallel.hpp:261-279). Over all cells
// of an axis this is A_a(lambda) = W_a^T diag(d_{lambda,a}) W_a with W_a
// lambda-free (rows s_m cos / s_m sin (2 pi m x), build_w
// symfourier.hpp:23-33). Summing spkmv over terms (parallel.hpp:184-228)
// therefore equals
//     psi = (W0^T (x) W1^T (x) W2^T) [ G .* ((W0 (x) W1 (x) W2) phi) ],
//     G[r0,r1,r2] = sum_lambda d_{l,0}[r0] d_{l,1}[r1] d_{l,2}[r2],
// which this file evaluates (rows compacted to R = 2M+1: the m=0 sine row of
// build_w is identically zero).
#include <cmath>

#include "internal.h"

namespace kb {
namespace {

// CellGrid::axis_nodes (geometry.hpp:102-110) minus the box centre
// (parallel.hpp:266-271), for mesh index x = cell * L + l.
__device__ __forceinline__ double mesh_node(const Geometry& g, int a, int x) {
    const int c = x / g.L, l = x % g.L;
    const double lo = g.center[a] - g.radius + 2.0 * g.radius * c / g.K[a];
    const double hi = g.center[a] - g.radius + 2.0 * g.radius * (c + 1) / g.K[a];
    return (lo + (hi - lo) * l / (g.L - 1)) - g.center[a];
}

// W_a[r][x], r = 0: m=0 cosine; r = 2m-1 / 2m: sqrt(2) cos / sin(2 pi m x).
__global__ void k_factor_w(Geometry g, int a, double* __restrict__ W) {
    const int n = g.n[a];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < g.R * n; e += gridDim.x * blockDim.x) {
        const int r = e / n, x = e % n;
        double v = 1.0;
        if (r > 0) {
            const int m = (r + 1) / 2;
            const double ph = 2.0 * M_PI * m * mesh_node(g, a, x);
            v = sqrt(2.0) * ((r & 1) ? cos(ph) : sin(ph));
        }
        W[e] = v;
    }
}

// D[t][a][r] = cbrt(weight_t) * even_profile(p_{t,a}, m(r))  (symfourier.hpp:69-71, 113-121)
__global__ void k_factor_d(Geometry g, int nterms, const double* __restrict__ tw,
                           const double* __restrict__ prof, double* __restrict__ D) {
    const int P = 2 * g.M + 1, R = g.R;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nterms * 3 * R;
         e += gridDim.x * blockDim.x) {
        const int t = e / (3 * R), a = (e / R) % 3, r = e % R, m = (r + 1) / 2;
        const double* p = prof + ((int64_t)t * 3 + a) * P;
        D[e] = cbrt(tw[t]) * (0.5 * (p[m + g.M] + p[g.M - m]));
    }
}

// G[r0][r1][r2] = sum_t D[t][0][r0] D[t][1][r1] D[t][2][r2], t ascending.
__global__ void k_factor_g(Geometry g, int nterms, const double* __restrict__ D,
                           double* __restrict__ G) {
    const int R = g.R;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * R * R;
         e += gridDim.x * blockDim.x) {
        const int r0 = e / (R * R), r1 = (e / R) % R, r2 = e % R;
        double s = 0.0;
        for (int t = 0; t < nterms; ++t) {
            const double* d = D + (int64_t)t * 3 * R;
            s = fma(d[r0] * d[R + r1], d[2 * R + r2], s);
        }
        G[e] = s;
    }
}

// Deterministic block sum of v[0..n): fixed per-thread strides, fixed tree.
__device__ double block_sum(const double* __restrict__ v, int n, double* red) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    return red[0];
}

// T2[x][r1][r2] = sum_y W1[r1][y] * sum_seg T1[seg][x][y][r2]
// All operands staged in shared memory first (coalesced, loads in flight).
__global__ void k_core_a(Geometry g, int S, const double* __restrict__ T1,
                         const double* __restrict__ W1, double* __restrict__ T2) {
    extern __shared__ double sh[];
    const int x = blockIdx.x, n1 = g.n[1], R = g.R;
    double* t1x = sh;             // n1 x R
    double* w1 = sh + n1 * R;     // R x n1
    const int64_t seg_stride = (int64_t)g.n[0] * n1 * R;
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
        double s = 0.0;
        for (int seg = 0; seg < S; ++seg) s += T1[seg * seg_stride + (int64_t)x * n1 * R + e];
        t1x[e] = s;
        w1[e] = W1[e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int r1 = e / R, r2 = e % R;
        double s = 0.0;
        for (int y = 0; y < n1; ++y) s = fma(w1[r1 * n1 + y], t1x[y * R + r2], s);
        T2[(int64_t)x * R * R + e] = s;
    }
}

// F[r0][e] = sum_x W0[r0][x] T2[x][e]; one CTA per (r0, e-chunk of 32):
// each warp reduces a strided slice of x, warps combined in a fixed order.
// F[R^3] = sum q (columns in order).
__global__ void k_core_b(Geometry g, int S, const double* __restrict__ T2,
                         const double* __restrict__ W0, const double* __restrict__ colq,
                         double* __restrict__ F) {
    __shared__ double part[8][32];
    __shared__ double red[256];
    const int R = g.R, RR = R * R, n0 = g.n[0];
    const int r0 = blockIdx.x, e = blockIdx.y * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
    double s = 0.0;
    if (e < RR)
        for (int x = w; x < n0; x += 8) s = fma(W0[(int64_t)r0 * n0 + x], T2[(int64_t)x * RR + e], s);
    part[w][threadIdx.x & 31] = s;
    __syncthreads();
    if (w == 0 && e < RR) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += part[k][threadIdx.x];
        F[(int64_t)r0 * RR + e] = t;
    }
    if (r0 == 0 && blockIdx.y == 0) {
        const double q = block_sum(colq, S * g.K[0] * g.K[1], red);
        if (threadIdx.x == 0) F[R * RR] = q;
    }
}

// B2[x][y][r2] = sum_r1 W1[r1][y] sum_r0 W0[r0][x] G[r0,r1,r2] F[r0,r1,r2];
// corr = c_Lambda * sum q.
__global__ void k_core_c(Geometry g, const double* __restrict__ G, const double* __restrict__ F,
                         double correction, const double* __restrict__ W0,
                         const double* __restrict__ W1, double* __restrict__ B2,
                         double* __restrict__ corr) {
    extern __shared__ double sh[];
    const int x = blockIdx.x, R = g.R, RR = R * R, n0 = g.n[0], n1 = g.n[1];
    double* b1 = sh;            // R x R
    double* w1 = sh + RR;       // R x n1
    double* h = w1 + R * n1;    // R^3: G .* F
    double* w0 = h + RR * R;    // R
    for (int e = threadIdx.x; e < RR * R; e += blockDim.x) h[e] = G[e] * F[e];
    for (int e = threadIdx.x; e < R * n1; e += blockDim.x) w1[e] = W1[e];
    if (threadIdx.x < R) w0[threadIdx.x] = W0[(int64_t)threadIdx.x * n0 + x];
    __syncthreads();
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
        double s = 0.0;
        for (int r0 = 0; r0 < R; ++r0) s = fma(w0[r0], h[r0 * RR + e], s);
        b1[e] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
        const int y = e / R, r2 = e % R;
        double s = 0.0;
        for (int r1 = 0; r1 < R; ++r1) s = fma(w1[r1 * n1 + y], b1[r1 * R + r2], s);
        B2[(int64_t)x * n1 * R + e] = s;
    }
    if (x == 0 && threadIdx.x == 0) *corr = correction * F[R * RR];
}

// F[e] = sum_b Fpart[e][b] (entry-major partials): one warp per entry, lanes
// over blocks, fixed shuffle tree (deterministic).
__global__ void k_core_sum(int nblocks, int E, const double* __restrict__ Fpart,
                           double* __restrict__ F) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    pdl_trigger();  // the gather may become resident and load its tables
    pdl_wait();     // the spread's partial cores
    if (e >= E) return;
    const double* row = Fpart + (int64_t)e * nblocks;
    // lane sums blocks lane + 64k (s0) and lane + 32 + 64k (s1) in increasing
    // k; 8 rounds of loads are issued before they are added (latency-bound)
    double s0 = 0.0, s1 = 0.0;
    for (int b0 = lane; b0 < nblocks; b0 += 64 * 8) {
        double v0[8], v1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = b0 + 64 * u;
            v0[u] = b < nblocks ? __ldg(row + b) : 0.0;
            v1[u] = b + 32 < nblocks ? __ldg(row + b + 32) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s0 += v0[u];
            s1 += v1[u];
        }
    }
    double s = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) F[e] = s;
}

__global__ void k_charge_correction(Geometry g, int S, const double* __restrict__ colq,
                                    double correction, double* __restrict__ corr) {
    __shared__ double red[128];
    const double q = block_sum(colq, S * g.K[0] * g.K[1], red);
    if (threadIdx.x == 0) *corr = correction * q;
}

// WL[r][c L + m] = sum_i W[r][c L + i] Lam[i][m]: the factor rows in the
// monomial basis of each cell (w_i(t) = sum_m Lam[i][m] t^m).
__global__ void k_factor_wl(Geometry g, int a, const double* __restrict__ W,
                            const double* __restrict__ lam, double* __restrict__ WL) {
    const int n = g.n[a], L = g.L;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < g.R * n; e += gridDim.x * blockDim.x) {
        const int r = e / n, x = e % n, c = x / L, m = x % L;
        double s = 0.0;
        for (int i = 0; i < L; ++i) s = fma(W[(int64_t)r * n + c * L + i], lam[i * L + m], s);
        // r = 0 is the constant row: sum_i w_i(t) = 1 exactly (interpolation
        // reproduces constants), so its monomial row is exactly (1, 0, ..., 0)
        if (r == 0) s = m == 0 ? 1.0 : 0.0;
        WL[e] = s;
    }
}

// out[t][u][v] = sum_r W[r][u] D[t][a][r] W[r][v]  (dense A_a(lambda))
__global__ void k_axis_operands(Geometry g, int a, int nterms, const double* __restrict__ W,
                                const double* __restrict__ D, double* __restrict__ out) {
    const int n = g.n[a], R = g.R, u = blockIdx.x, t = blockIdx.y;
    const double* d = D + ((int64_t)t * 3 + a) * R;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < R; ++r) s = fma(W[(int64_t)r * n + u] * d[r], W[(int64_t)r * n + v], s);
        out[((int64_t)t * n + u) * n + v] = s;
    }
}

// per-cell grids [cell][L^3] <-> lexicographic mesh [n0][n1][n2]
__global__ void k_cells_mesh(Geometry g, const double* __restrict__ src, double* __restrict__ dst,
                             int inverse) {
    const int64_t total = (int64_t)g.n[0] * g.n[1] * g.n[2];
    const int L = g.L;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(e % g.n[2]);
        const int y = (int)((e / g.n[2]) % g.n[1]);
        const int x = (int)(e / ((int64_t)g.n[1] * g.n[2]));
        const int cell = ((x / L) * g.K[1] + y / L) * g.K[2] + z / L;
        const int64_t ci = (int64_t)cell * L * L * L + ((x % L) * L + y % L) * L + z % L;
        if (inverse)
            dst[ci] = src[e];
        else
            dst[e] = src[ci];
    }
}

}  // namespace

void launch_factor_tables(const Geometry& g, int nterms, const double* tw, const double* prof,
                          double* W0, double* W1, double* W2, double* D, double* G,
                          cudaStream_t s) {
    double* W[3] = {W0, W1, W2};
    for (int a = 0; a < 3; ++a) {
        k_factor_w<<<64, 256, 0, s>>>(g, a, W[a]);
        KB_CHECK_LAUNCH();
    }
    if (nterms > 0) {
        k_factor_d<<<16, 256, 0, s>>>(g, nterms, tw, prof, D);
        KB_CHECK_LAUNCH();
    }
    k_factor_g<<<16, 256, 0, s>>>(g, nterms, D, G);
    KB_CHECK_LAUNCH();
}

void launch_core_forward(const Geometry& g, int S, const double* T1, const double* W0,
                         const double* W1, double* T2, const double* colq, double* F,
                         cudaStream_t s) {
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_core_a, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_core_c, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
    });
    k_core_a<<<g.n[0], 128, sizeof(double) * 2 * g.n[1] * g.R, s>>>(g, S, T1, W1, T2);
    KB_CHECK_LAUNCH();
    k_core_b<<<dim3(g.R, (g.R * g.R + 31) / 32), 256, 0, s>>>(g, S, T2, W0, colq, F);
    KB_CHECK_LAUNCH();
}

void launch_core_backward(const Geometry& g, const double* G, const double* F, double correction,
                          const double* W0, const double* W1, double* B2, double* corr,
                          cudaStream_t s) {
    const size_t sh = sizeof(double) * ((size_t)g.R * g.R * (g.R + 1) + (size_t)g.R * g.n[1] + g.R);
    k_core_c<<<g.n[0], 256, sh, s>>>(g, G, F, correction, W0, W1, B2, corr);
    KB_CHECK_LAUNCH();
}

void launch_core_sum(const Geometry& g, int nblocks, const double* Fpart, double* F,
                     cudaStream_t s) {
    const int E = g.R * g.R * g.R + 1;
    launch_pdl_if((pdl_mask() & 4) != 0, k_core_sum, dim3((E + 7) / 8), dim3(256), 0, s, nblocks, E, Fpart, F);
    KB_CHECK_LAUNCH();
}

void launch_charge_correction(const Geometry& g, int S, const double* colq, double correction,
                              double* corr, cudaStream_t s) {
    k_charge_correction<<<1, 128, 0, s>>>(g, S, colq, correction, corr);
    KB_CHECK_LAUNCH();
}

void launch_factor_wl(const Geometry& g, int axis, const double* W, const double* lam, double* WL,
                      cudaStream_t s) {
    k_factor_wl<<<64, 256, 0, s>>>(g, axis, W, lam, WL);
    KB_CHECK_LAUNCH();
}

void launch_axis_operands(const Geometry& g, int a, int nterms, const double* W, const double* D,
                          double* out, cudaStream_t s) {
    if (nterms <= 0) return;
    k_axis_operands<<<dim3(g.n[a], nterms), 128, 0, s>>>(g, a, nterms, W, D, out);
    KB_CHECK_LAUNCH();
}

void launch_cells_to_mesh(const Geometry& g, const double* src, double* dst, bool inverse,
                          cudaStream_t s) {
    k_cells_mesh<<<sm_count() * 8, 256, 0, s>>>(g, src, dst, inverse ? 1 : 0);
    KB_CHECK_LAUNCH();
}

}  // namespace kb
