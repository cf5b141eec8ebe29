// Shared-memory load throughput on B200 for the gather's coefficient reads:
// 64-bit and 128-bit loads, all lanes reading the same address (broadcast)
// or distinct addresses. 16 warps/SM, cycles per warp-instruction per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters) {
    __shared__ __align__(16) double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 1e-3;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int base = (threadIdx.x >> 5) * 64;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int off = (base + u * 2) & 4094;
            if (MODE == 0) {  // LDS.64 broadcast
                acc0 += s[off]; acc1 += s[off + 1];
            } else if (MODE == 1) {  // LDS.128 broadcast
                const double2 v = *reinterpret_cast<const double2*>(s + off);
                acc0 += v.x; acc1 += v.y;
            } else if (MODE == 2) {  // LDS.64 distinct (lane stride 1)
                acc0 += s[(off + lane) & 4095]; acc1 += s[(off + lane + 32) & 4095];
            } else {  // LDS.128 distinct
                const double2 v = *reinterpret_cast<const double2*>(s + ((off + 2 * lane) & 4094));
                acc0 += v.x; acc1 += v.y;
            }
        }
        base += 32;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 512 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4000;
    const char* names[4] = {"LDS.64 broadcast (2 per 16B)", "LDS.128 broadcast", "LDS.64 distinct (2 per 16B)", "LDS.128 distinct"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148, 512>>>(out, iters);
            if (mode == 1) k<1><<<148, 512>>>(out, iters);
            if (mode == 2) k<2><<<148, 512>>>(out, iters);
            if (mode == 3) k<3><<<148, 512>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            int clk;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            const double cycles = ms * 1e-3 * clk * 1e3;
            const double loads16 = 16.0 * iters * 16;  // 16-byte fetches per warp... per SM: 16 warps
            if (rep) printf("%-30s %.3f ms  %.2f SM-cycles per 16B-per-lane warp fetch\n", names[mode], ms, cycles / loads16);
        }
    }
    return 0;
}
