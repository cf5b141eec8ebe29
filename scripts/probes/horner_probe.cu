// Horner-gather inner loop probe (sm_100a): NCH particle chains per lane
// evaluated against an L^3 coefficient block in shared memory, as in
// k_gather_cc; reports FMA/clk/SM at 1..4 warps per SM sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int L = 6;
template <int NCH, int ROLL, int MODE>
__global__ void k_horner(int iters, double* out, long long* cycles) {
    __shared__ __align__(16) double psi[4 * L * L * L];
    for (int e = threadIdx.x; e < 4 * L * L * L; e += blockDim.x) psi[e] = 1e-3 * e;
    double t0[NCH], t1[NCH], t2[NCH], z[NCH], acc[NCH];
    for (int u = 0; u < NCH; ++u) {
        t0[u] = 0.1 * threadIdx.x + u;
        t1[u] = 0.2 * threadIdx.x - u;
        t2[u] = 0.3 + u;
        acc[u] = 0;
    }
    const double creg = psi[threadIdx.x & 7];
    __syncthreads();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double* ps = psi + (it & 3) * L * L * L;
        for (int u = 0; u < NCH; ++u) z[u] = 0.0;
#pragma unroll ROLL
        for (int i = L - 1; i >= 0; --i) {
            double zb[NCH];
#pragma unroll
            for (int j = L - 1; j >= 0; --j) {
                const double* row = ps + (i * L + j) * L;
                double c[L];
if (MODE == 0) {
#pragma unroll
                for (int k = 0; k < L; k += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(row + k);
                    c[k] = v.x;
                    c[k + 1] = v.y;
                }
                } else if (MODE == 2) {
#pragma unroll
                for (int k = 0; k < L; ++k) c[k] = row[k];
                } else {
#pragma unroll
                for (int k = 0; k < L; ++k) c[k] = creg + (double)(i * 36 + j * 6 + k);
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
        for (int u = 0; u < NCH; ++u) {
            acc[u] += z[u];
            t2[u] += 1e-9 * z[u];
        }
    }
    const long long c1 = clock64();
    double s = 0;
    for (int u = 0; u < NCH; ++u) s += acc[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
}
template <int NCH, int ROLL, int MODE>
void run(int warps, double* out, long long* cyc) {
    const int iters = 512;
    k_horner<NCH, ROLL, MODE><<<148, 32 * warps>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double fmas = (double)iters * NCH * (L * L * L - 1) * 32.0 * warps;
    printf("chains=%d roll=%d mode=%d warps/SM=%2d: %5.1f FMA/clk/SM\n", NCH, ROLL, MODE, warps, fmas / (double)h);
}
int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8);
    for (int w : {4, 8, 12}) {
        run<4, 1, 0>(w, out, cyc);
        run<4, 1, 2>(w, out, cyc);
        run<4, 1, 1>(w, out, cyc);
        run<4, 6, 1>(w, out, cyc);
        run<6, 1, 0>(w, out, cyc);
        run<8, 1, 0>(w, out, cyc);
        run<2, 1, 0>(w, out, cyc);
        run<2, 1, 1>(w, out, cyc);
    }
    return 0;
}
