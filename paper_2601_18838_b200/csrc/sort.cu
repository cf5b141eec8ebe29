// sort.cu -- bit-exact cell sort (assign_particles, geometry.hpp:131-154).
//
// Pipeline: cell key + box check + histogram (integer atomics only) ->
// exclusive scan -> scatter into cell segments -> per-cell sort of the
// member indices. The last step restores the reference's "ascending particle
// index within each cell" order (Partition.members, geometry.hpp:124-127), so
// the result is identical to the reference whatever order the atomics ran in.
#include <climits>

#include "internal.h"

namespace kb {
namespace {

constexpr int kWarpCap = 1024;      // largest segment sorted by one warp
constexpr int kBlockCap = 16384;    // largest segment sorted by one CTA in smem

// Cell index along one axis, in the reference's exact operation order
// (geometry.hpp:141-148). Explicit round-to-nearest intrinsics: no FMA
// contraction may change a bit of t.
__device__ __forceinline__ int axis_cell(double p, double c, double r, int K) {
    const double t = __ddiv_rn(__dmul_rn(__dsub_rn(p, __dsub_rn(c, r)), (double)K),
                               __dmul_rn(2.0, r));
    int idx = (int)floor(t);
    if (t == (double)idx && idx > 0) --idx;
    if (idx < 0) idx = 0;
    if (idx > K - 1) idx = K - 1;
    return idx;
}

__global__ void k_keys(Geometry g, int64_t n, const double* __restrict__ xyz,
                       int32_t* __restrict__ key, int32_t* __restrict__ cnt,
                       unsigned long long* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double p0 = xyz[3 * i], p1 = xyz[3 * i + 1], p2 = xyz[3 * i + 2];
        // Box3::contains (geometry.hpp:36-40)
        if (fabs(p0 - g.center[0]) > g.radius || fabs(p1 - g.center[1]) > g.radius ||
            fabs(p2 - g.center[2]) > g.radius)
            atomicMin(&bad[0], (unsigned long long)i);
        const int c0 = axis_cell(p0, g.center[0], g.radius, g.K[0]);
        const int c1 = axis_cell(p1, g.center[1], g.radius, g.K[1]);
        const int c2 = axis_cell(p2, g.center[2], g.radius, g.K[2]);
        if (c2 < g.z_lo || c2 >= g.z_hi) atomicOr(&bad[1], 2ull);  // not in this slab
        const int k = (c0 * g.K[1] + c1) * g.K[2] + c2;  // CellGrid::flatten
        key[i] = k;
        atomicAdd(&cnt[k], 1);
    }
}

// Exclusive scan of the histogram by one CTA; leaves start[] and resets cnt[]
// to the running cursor.
__global__ void k_scan(int ncell, int32_t* __restrict__ cnt, int32_t* __restrict__ start) {
    __shared__ int32_t wsum[32];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int per = (ncell + T - 1) / T;
    const int b = min(tid * per, ncell), e = min(b + per, ncell);
    int local = 0;
    for (int i = b; i < e; ++i) local += cnt[i];
    int x = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int v = lane < (T >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    int run = x - local + (w > 0 ? wsum[w - 1] : 0);
    for (int i = b; i < e; ++i) {
        const int c = cnt[i];
        start[i] = run;
        cnt[i] = run;
        run += c;
    }
    if (tid == T - 1) start[ncell] = run;
}

__global__ void k_scatter(int64_t n, const int32_t* __restrict__ key, int32_t* cursor,
                          int32_t* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        perm[atomicAdd(&cursor[key[i]], 1)] = (int32_t)i;
}

// One warp per cell: restore ascending member order.
__global__ void __launch_bounds__(256) k_segsort_warp(int ncell, const int32_t* __restrict__ start,
                                                      int32_t* __restrict__ perm,
                                                      int32_t* __restrict__ big,
                                                      int32_t* __restrict__ nbig) {
    __shared__ int32_t buf[8][kWarpCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * 8 + w;
    if (cell >= ncell) return;
    const int s0 = start[cell], cnt = start[cell + 1] - s0;
    if (cnt <= 1) return;
    if (cnt > kWarpCap) {
        if (lane == 0) big[atomicAdd(nbig, 1)] = cell;
        return;
    }
    if (cnt <= 32) {  // register bitonic network across the warp
        int v = lane < cnt ? perm[s0 + lane] : INT_MAX;
        for (int k = 2; k <= 32; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                const int o = __shfl_xor_sync(0xffffffffu, v, j);
                const bool up = (lane & k) == 0, lower = (lane & j) == 0;
                v = (lower == up) ? min(v, o) : max(v, o);
            }
        if (lane < cnt) perm[s0 + lane] = v;
        return;
    }
    int P = 64;
    while (P < cnt) P <<= 1;
    int32_t* b = buf[w];
    for (int i = lane; i < P; i += 32) b[i] = i < cnt ? perm[s0 + i] : INT_MAX;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const int x = b[i], y = b[ixj];
                    if ((x > y) == up) {
                        b[i] = y;
                        b[ixj] = x;
                    }
                }
            }
            __syncwarp();
        }
    for (int i = lane; i < cnt; i += 32) perm[s0 + i] = b[i];
}

// Large cells: one CTA per cell. Up to kBlockCap members are sorted in shared
// memory; beyond that the CTA rebuilds the segment by a stable, in-order
// compaction over all keys (O(n) per huge cell, only for degenerate inputs).
__global__ void __launch_bounds__(1024) k_segsort_big(int64_t n, const int32_t* __restrict__ key,
                                                      const int32_t* __restrict__ start,
                                                      int32_t* __restrict__ perm,
                                                      const int32_t* __restrict__ big,
                                                      const int32_t* __restrict__ nbig) {
    extern __shared__ int32_t sbuf[];
    __shared__ int32_t wcount[32];
    __shared__ int32_t offset;
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, w = tid >> 5;
    const int nb = *nbig;
    for (int bi = blockIdx.x; bi < nb; bi += gridDim.x) {
        const int cell = big[bi];
        const int s0 = start[cell], cnt = start[cell + 1] - s0;
        if (cnt <= kBlockCap) {
            int P = 1;
            while (P < cnt) P <<= 1;
            for (int i = tid; i < P; i += T) sbuf[i] = i < cnt ? perm[s0 + i] : INT_MAX;
            __syncthreads();
            for (int k = 2; k <= P; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = tid; i < P; i += T) {
                        const int ixj = i ^ j;
                        if (ixj > i) {
                            const bool up = (i & k) == 0;
                            const int x = sbuf[i], y = sbuf[ixj];
                            if ((x > y) == up) {
                                sbuf[i] = y;
                                sbuf[ixj] = x;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int i = tid; i < cnt; i += T) perm[s0 + i] = sbuf[i];
            __syncthreads();
        } else {
            if (tid == 0) offset = 0;
            __syncthreads();
            for (int64_t base = 0; base < n; base += T) {
                const int64_t i = base + tid;
                const bool hit = i < n && key[i] == cell;
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (lane == 0) wcount[w] = __popc(m);
                __syncthreads();
                int before = offset;
                for (int k = 0; k < w; ++k) before += wcount[k];
                if (hit) perm[s0 + before + __popc(m & ((1u << lane) - 1))] = (int32_t)i;
                __syncthreads();
                if (tid == 0) {
                    int tot = 0;
                    for (int k = 0; k < (T >> 5); ++k) tot += wcount[k];
                    offset += tot;
                }
                __syncthreads();
            }
        }
    }
}

__global__ void k_permute(int64_t n, const double* __restrict__ xyz, const double* __restrict__ q,
                          const int32_t* __restrict__ perm, double4* __restrict__ sp) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = perm[s];
        sp[s] = make_double4(xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2], q[p]);
    }
}

int grid_for(int64_t n, int threads) {
    const int64_t b = (n + threads - 1) / threads;
    return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

void launch_sort(const Geometry& g, int64_t n, const double* xyz, const SortBuffers& b,
                 cudaStream_t s, int* launches) {
    static bool attr_set = false;
    if (!attr_set) {
        KB_CUDA(cudaFuncSetAttribute(k_segsort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBlockCap * (int)sizeof(int32_t)));
        attr_set = true;
    }
    KB_CUDA(cudaMemsetAsync(b.cnt, 0, sizeof(int32_t) * g.ncell, s));
    KB_CUDA(cudaMemsetAsync(b.nbig, 0, sizeof(int32_t), s));
    if (n > 0) {
        k_keys<<<grid_for(n, 256), 256, 0, s>>>(g, n, xyz, b.key, b.cnt, b.bad);
        KB_CHECK_LAUNCH();
    }
    k_scan<<<1, 1024, 0, s>>>(g.ncell, b.cnt, b.start);
    KB_CHECK_LAUNCH();
    int l = 2;
    if (n > 0) {
        k_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, b.key, b.cnt, b.perm);
        KB_CHECK_LAUNCH();
        k_segsort_warp<<<(g.ncell + 7) / 8, 256, 0, s>>>(g.ncell, b.start, b.perm, b.big, b.nbig);
        KB_CHECK_LAUNCH();
        k_segsort_big<<<148, 1024, kBlockCap * sizeof(int32_t), s>>>(n, b.key, b.start, b.perm,
                                                                    b.big, b.nbig);
        KB_CHECK_LAUNCH();
        l += 4;
    }
    if (launches) *launches += l;
}

void launch_permute(int64_t n, const double* xyz, const double* q, const int32_t* perm,
                    double4* sp, cudaStream_t s) {
    if (n <= 0) return;
    k_permute<<<grid_for(n, 256), 256, 0, s>>>(n, xyz, q, perm, sp);
    KB_CHECK_LAUNCH();
}

}  // namespace kb
