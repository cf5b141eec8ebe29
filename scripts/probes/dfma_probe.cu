// DFMA latency / throughput probe (sm_100a): cycles per DFMA warp-instruction
// for 1..12 independent chains per warp at 1, 2, 3 and 4 warps per SM
// sub-partition, plus the same with an operand read from shared memory.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, bool LDS>
__global__ void k_dfma(int iters, double* out, long long* cycles) {
    __shared__ double coef[64];
    if (threadIdx.x < 64) coef[threadIdx.x] = 0.5 + threadIdx.x * 1e-3;
    double c[CHAINS];
    for (int i = 0; i < CHAINS; ++i) c[i] = threadIdx.x + i;
    const double t = 1.0000001;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double k = LDS ? coef[it & 63] : 0.5;
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], t, k);
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CHAINS, bool LDS>
void run(int warps, double* out, long long* cyc) {
    const int iters = 8192;
    k_dfma<CHAINS, LDS><<<148, 32 * warps>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double per = (double)h / ((double)iters * CHAINS);
    printf("chains=%2d lds=%d warps/SM=%2d: %6.2f cyc per DFMA per warp -> %5.1f FMA/clk/SM\n", CHAINS, (int)LDS,
           warps, per, 32.0 * warps / per);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8);
    for (int w : {4, 8, 12, 16}) {
        run<1, false>(w, out, cyc);
        run<2, false>(w, out, cyc);
        run<4, false>(w, out, cyc);
        run<6, false>(w, out, cyc);
        run<8, false>(w, out, cyc);
        run<12, false>(w, out, cyc);
        run<4, true>(w, out, cyc);
        run<8, true>(w, out, cyc);
    }
    return 0;
}
