// sort.cu -- bit-exact cell sort (assign_particles, geometry.hpp:131-154).
//
// Pipeline: cell key + box check + histogram whose atomic also hands each
// particle a provisional slot in its cell (integer atomics only) -> exclusive
// scan -> placement into cell segments -> per-cell sort of the member indices. The last step restores the reference's "ascending particle
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
                       int32_t* __restrict__ key, int32_t* __restrict__ rank,
                       int32_t* __restrict__ cnt, unsigned long long* bad) {
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
        rank[i] = atomicAdd(&cnt[k], 1);  // provisional slot, fixed up by k_segsort
    }
}

// Exclusive scan of the histogram by one CTA, in shared-memory chunks of
// kScanChunk counts (coalesced loads, all in flight); leaves start[] and
// resets cnt[] to the running cursor.
constexpr int kScanChunk = 16384;
__global__ void __launch_bounds__(1024) k_scan(int ncell, int32_t* __restrict__ cnt,
                                               int32_t* __restrict__ start) {
    extern __shared__ int32_t sc[];  // kScanChunk
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr int per = kScanChunk / 1024;
    if (tid == 0) carry = 0;
    for (int base = 0; base < ncell; base += kScanChunk) {
        const int m = min(kScanChunk, ncell - base);
        for (int i = tid; i < kScanChunk; i += T) sc[i] = i < m ? cnt[base + i] : 0;
        __syncthreads();
        int local = 0;
#pragma unroll
        for (int k = 0; k < per; ++k) local += sc[tid * per + k];
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
        int run = carry + x - local + (w > 0 ? wsum[w - 1] : 0);
#pragma unroll
        for (int k = 0; k < per; ++k) {
            const int c = sc[tid * per + k];
            sc[tid * per + k] = run;
            run += c;
        }
        __syncthreads();
        for (int i = tid; i < m; i += T) {
            start[base + i] = sc[i];
            cnt[base + i] = sc[i];
        }
        if (tid == T - 1) carry = run;
        __syncthreads();
    }
    if (tid == 0) start[ncell] = carry;
}

__global__ void k_place(int64_t n, const int32_t* __restrict__ key,
                        const int32_t* __restrict__ rank, const int32_t* __restrict__ start,
                        int32_t* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        perm[start[key[i]] + rank[i]] = (int32_t)i;
}

// sorted particle record for slot s (fused permute)
__device__ __forceinline__ void put_sp(double4* sp, const double* __restrict__ xyz,
                                       const double* __restrict__ q, int64_t slot, int32_t v) {
    if (sp) sp[slot] = make_double4(xyz[3 * (int64_t)v], xyz[3 * (int64_t)v + 1],
                                    xyz[3 * (int64_t)v + 2], q[v]);
}

// Warp rank sort of b[0..cnt) (distinct values, padded to P4 with INT_MAX):
// member k of lane l goes to out[number of smaller members].
template <int V>
__device__ __forceinline__ void rank_sort(const int32_t* b, int P4, int cnt, int lane,
                                          int32_t* out, double4* sp, const double* xyz,
                                          const double* q) {
    int v[V], r[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        v[k] = (lane + 32 * k < cnt) ? b[lane + 32 * k] : INT_MAX;
        r[k] = 0;
    }
    for (int j = 0; j < P4; j += 4) {
        const int4 x = *reinterpret_cast<const int4*>(b + j);
#pragma unroll
        for (int k = 0; k < V; ++k) r[k] += (x.x < v[k]) + (x.y < v[k]) + (x.z < v[k]) + (x.w < v[k]);
    }
#pragma unroll
    for (int k = 0; k < V; ++k)
        if (lane + 32 * k < cnt) {
            out[r[k]] = v[k];
            put_sp(sp, xyz, q, r[k], v[k]);
        }
}

// One warp per cell: restore ascending member order.
__global__ void __launch_bounds__(256) k_segsort_warp(int ncell, const int32_t* __restrict__ start,
                                                      int32_t* __restrict__ perm,
                                                      int32_t* __restrict__ big,
                                                      int32_t* __restrict__ nbig,
                                                      const double* __restrict__ xyz,
                                                      const double* __restrict__ q,
                                                      double4* __restrict__ sp) {
    __shared__ __align__(16) int32_t buf[8][kWarpCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * 8 + w;
    if (cell >= ncell) return;
    const int s0 = start[cell], cnt = start[cell + 1] - s0;
    if (cnt == 0) return;
    if (cnt == 1) {
        if (lane == 0) put_sp(sp, xyz, q, s0, perm[s0]);
        return;
    }
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
        if (lane < cnt) {
            perm[s0 + lane] = v;
            put_sp(sp, xyz, q, s0 + lane, v);
        }
        return;
    }
    int32_t* b = buf[w];
    if (cnt <= 256) {
        // rank by counting: each member's slot = number of smaller members
        const int P4 = (cnt + 3) & ~3;
        for (int i = lane; i < P4; i += 32) b[i] = i < cnt ? perm[s0 + i] : INT_MAX;
        __syncwarp();
        double4* sps = sp ? sp + s0 : nullptr;
        if (cnt <= 128) rank_sort<4>(b, P4, cnt, lane, perm + s0, sps, xyz, q);
        else rank_sort<8>(b, P4, cnt, lane, perm + s0, sps, xyz, q);
        return;
    }
    int P = 512;
    while (P < cnt) P <<= 1;
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
    for (int i = lane; i < cnt; i += 32) {
        perm[s0 + i] = b[i];
        put_sp(sp, xyz, q, s0 + i, b[i]);
    }
}

// Large cells: one CTA per cell. Up to kBlockCap members are sorted in shared
// memory; beyond that the CTA rebuilds the segment by a stable, in-order
// compaction over all keys (O(n) per huge cell, only for degenerate inputs).
__global__ void __launch_bounds__(1024) k_segsort_big(int64_t n, const int32_t* __restrict__ key,
                                                      const int32_t* __restrict__ start,
                                                      int32_t* __restrict__ perm,
                                                      const int32_t* __restrict__ big,
                                                      const int32_t* __restrict__ nbig,
                                                      const double* __restrict__ xyz,
                                                      const double* __restrict__ q,
                                                      double4* __restrict__ sp) {
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
            for (int i = tid; i < cnt; i += T) {
                perm[s0 + i] = sbuf[i];
                put_sp(sp, xyz, q, s0 + i, sbuf[i]);
            }
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
            if (sp) {
                __threadfence_block();
                for (int i = tid; i < cnt; i += T) put_sp(sp, xyz, q, s0 + i, perm[s0 + i]);
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
                 cudaStream_t s, int* launches, const double* q, double4* sp) {
    if (!q) sp = nullptr;
    static bool attr_set = false;
    if (!attr_set) {
        KB_CUDA(cudaFuncSetAttribute(k_segsort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBlockCap * (int)sizeof(int32_t)));
        KB_CUDA(cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kScanChunk * (int)sizeof(int32_t)));
        attr_set = true;
    }
    KB_CUDA(cudaMemsetAsync(b.cnt, 0, sizeof(int32_t) * g.ncell, s));
    KB_CUDA(cudaMemsetAsync(b.nbig, 0, sizeof(int32_t), s));
    if (n > 0) {
        k_keys<<<grid_for(n, 256), 256, 0, s>>>(g, n, xyz, b.key, b.rank, b.cnt, b.bad);
        KB_CHECK_LAUNCH();
    }
    k_scan<<<1, 1024, kScanChunk * sizeof(int32_t), s>>>(g.ncell, b.cnt, b.start);
    KB_CHECK_LAUNCH();
    int l = 2;
    if (n > 0) {
        k_place<<<grid_for(n, 256), 256, 0, s>>>(n, b.key, b.rank, b.start, b.perm);
        KB_CHECK_LAUNCH();
        k_segsort_warp<<<(g.ncell + 7) / 8, 256, 0, s>>>(g.ncell, b.start, b.perm, b.big, b.nbig,
                                                         xyz, q, sp);
        KB_CHECK_LAUNCH();
        k_segsort_big<<<148, 1024, kBlockCap * sizeof(int32_t), s>>>(n, b.key, b.start, b.perm,
                                                                    b.big, b.nbig, xyz, q, sp);
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
