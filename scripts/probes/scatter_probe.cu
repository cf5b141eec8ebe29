// Calibration probe: cost of scattered / gathered record moves on B200.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scatter_probe.cu -o scatter_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void copy4(const double4* __restrict__ a, double4* __restrict__ b, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}
__global__ void scatter4(const double4* __restrict__ a, const int* __restrict__ p, double4* __restrict__ b, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[p[i]] = a[i];
}
__global__ void gather4(const double4* __restrict__ a, const int* __restrict__ p, double4* __restrict__ b, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[p[i]];
}
__global__ void scatter1(const int* __restrict__ a, const int* __restrict__ p, int* __restrict__ b, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[p[i]] = a[i];
}
__global__ void flush(float* f, size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = f[i] * 0.5f + 1.f;
}

int main() {
    const int n = 1 << 20;
    std::mt19937 rng(1);
    std::vector<int> perm(n), local(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), rng);
    // windowed: random positions inside windows of 2268 (a cell column)
    const int W = 2268;
    for (int s = 0; s < n; s += W) {
        int e = std::min(n, s + W);
        std::vector<int> w(e - s);
        for (int i = 0; i < e - s; ++i) w[i] = s + i;
        std::shuffle(w.begin(), w.end(), rng);
        for (int i = s; i < e; ++i) local[i] = w[i - s];
    }
    // tile->column scatter pattern: 441 columns, stable by tile
    std::vector<int> colp(n);
    {
        std::vector<int> col(n), cnt(441, 0), off(441, 0);
        for (int i = 0; i < n; ++i) { col[i] = rng() % 441; cnt[col[i]]++; }
        for (int c = 1; c < 441; ++c) off[c] = off[c - 1] + cnt[c - 1];
        for (int i = 0; i < n; ++i) colp[i] = off[col[i]]++;
    }
    double4 *a, *b; int *p, *pl, *pc, *ia, *ib; float* f;
    cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32); cudaMalloc(&p, n * 4); cudaMalloc(&pl, n * 4);
    cudaMalloc(&pc, n * 4); cudaMalloc(&ia, n * 4); cudaMalloc(&ib, n * 4);
    size_t fn = 64u << 20; cudaMalloc(&f, fn * 4);
    cudaMemset(a, 0, n * 32);
    cudaMemcpy(p, perm.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(pl, local.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(pc, colp.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, bool warm) {
        float best = 1e9, sum = 0;
        for (int r = 0; r < 10; ++r) {
            if (!warm) flush<<<592, 1024>>>(f, fn);
            else launch();
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); sum += ms;
        }
        printf("%-28s %s best %7.2f us  avg %7.2f us\n", name, warm ? "warm" : "cold", best * 1e3, sum * 100);
    };
    const int T = 256, G = (n + T - 1) / T;
    for (int warm = 0; warm < 2; ++warm) {
        run("copy double4", [&] { copy4<<<G, T>>>(a, b, n); }, warm);
        run("scatter double4 random", [&] { scatter4<<<G, T>>>(a, p, b, n); }, warm);
        run("gather double4 random", [&] { gather4<<<G, T>>>(a, p, b, n); }, warm);
        run("scatter double4 window2268", [&] { scatter4<<<G, T>>>(a, pl, b, n); }, warm);
        run("gather double4 window2268", [&] { gather4<<<G, T>>>(a, pl, b, n); }, warm);
        run("scatter double4 441cols", [&] { scatter4<<<G, T>>>(a, pc, b, n); }, warm);
        run("scatter int random", [&] { scatter1<<<G, T>>>(ia, p, ib, n); }, warm);
        run("scatter int 441cols", [&] { scatter1<<<G, T>>>(ia, pc, ib, n); }, warm);
    }
    return 0;
}
