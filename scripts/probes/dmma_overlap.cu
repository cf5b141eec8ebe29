// Does DMMA on one warp overlap with FP64 / integer work of another warp on
// the same SM sub-partition? Warps 0 and 4 of a 8-warp CTA share SMSP 0.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_overlap.cu -o dmma_overlap
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void k(int mode, int iters, double* out, long long* cyc) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc[8][2] = {};
    double x = lane * 1e-3, y = 1.0 + lane * 1e-4;
    long long t0 = clock64();
    if (w == 0 && (mode & 1)) {  // DMMA stream: 8 independent chains
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int t = 0; t < 8; ++t) dmma(acc[t], x, y);
    }
    if (w == 4 && (mode & 2)) {  // DFMA stream: 8 independent chains
        double z[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) z[t] = x + t;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int t = 0; t < 8; ++t) z[t] = fma(z[t], y, x);
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t][0] += z[t];
    }
    if (w == 4 && (mode & 4)) {  // integer / shared-memory stream
        __shared__ int sh[256];
        int v = lane;
        for (int i = 0; i < iters * 8; ++i) {
            v = v * 1664525 + 1013904223;
            sh[(v >> 8) & 255] = v;
        }
        acc[0][0] += sh[lane];
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += acc[t][0] + acc[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (lane == 0) cyc[blockIdx.x * 8 + w] = t1 - t0;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 256 * 8);
    cudaMalloc(&cyc, 148 * 8 * 8);
    long long h[8];
    const int iters = 2000;
    const char* names[] = {"", "dmma only", "dfma only", "dmma+dfma", "int/smem only", "dmma+int/smem"};
    for (int mode : {1, 2, 3, 4, 5}) {
        k<<<148, 256>>>(mode, iters, out, cyc);
        cudaDeviceSynchronize();
        k<<<148, 256>>>(mode, iters, out, cyc);
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-16s warp0 %8lld cycles  warp4 %8lld cycles\n", names[mode], h[0], h[4]);
    }
    return 0;
}
