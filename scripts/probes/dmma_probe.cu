// DMMA.8x8x4 latency / throughput probe (sm_100a). Prints cycles per DMMA
// for a dependent chain and for k independent accumulators, and the SM-wide
// FP64 tensor rate with many warps.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void k_probe(int iters, double* out, long long* cycles) {
    double c[CHAINS][2];
    for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i;
    const double a = 1.0000001, b = 0.9999999;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) dmma(c[i], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(int iters, double* out, long long* cycles) {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x + i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(c[i], 1.0000001, 0.5);
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CHAINS>
void run(const char* name, int warps_per_block, int blocks, int iters, double* out, long long* cyc) {
    k_probe<CHAINS><<<blocks, 32 * warps_per_block>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double per = (double)h / ((double)iters * CHAINS);
    const double per_sm_warps = (double)warps_per_block * (blocks >= 148 ? blocks / 148.0 : 1.0);
    printf("%-34s warps/blk=%2d blocks=%4d : %7.2f cyc per DMMA per warp -> %6.1f FMA/clk/SM\n", name,
           warps_per_block, blocks, per, 256.0 * per_sm_warps / per);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 8 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8 * 8);
    const int iters = 4096;
    run<1>("dependent chain (1 acc)", 1, 1, iters, out, cyc);
    run<2>("2 accumulators", 1, 1, iters, out, cyc);
    run<4>("4 accumulators", 1, 1, iters, out, cyc);
    run<8>("8 accumulators", 1, 1, iters, out, cyc);
    run<16>("16 accumulators", 1, 1, iters, out, cyc);
    run<8>("8 acc, 4 warps/SM", 4, 148, iters, out, cyc);
    run<8>("8 acc, 8 warps/SM", 8, 148, iters, out, cyc);
    run<8>("8 acc, 16 warps/SM", 16, 148, iters, out, cyc);
    run<2>("2 acc, 16 warps/SM", 16, 148, iters, out, cyc);
    run<5>("5 acc, 12 warps/SM", 12, 148, iters, out, cyc);
    k_dfma<<<148, 512>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("DFMA, 16 warps/SM, 8 chains: %.2f cyc per DFMA-instr per warp -> %.1f FMA/clk/SM\n",
           (double)h / (iters * 8.0), 32.0 * 16 / ((double)h / (iters * 8.0)));
    return 0;
}
