// sort.cu -- bit-exact cell sort (assign_particles, geometry.hpp:131-154)
// fused with the construction of the cell-ordered particle records.
//
//   k_keys    cell key in the reference's exact arithmetic + box check; the
//             histogram atomic also hands out a provisional slot in the cell
//   k_scan    exclusive scan of the histogram -> cell_start
//   k_place   perm[start + slot] = i and, with charges, the packed record
//             (x, y, z, q) at the same provisional slot (coalesced reads,
//             one 32-byte sector written per particle)
//   k_segsort per cell: restore the reference's ascending-index member order
//             (Partition.members, geometry.hpp:124-127) and move the records
//             inside the cell's contiguous segment
// The result is identical to the reference whatever order the atomics ran in.
#include <climits>

#include "internal.h"

namespace kb {
namespace {

constexpr int kRankCap = 256;      // warp rank-count sort
constexpr int kWarpCap = 512;      // warp bitonic sort of (index, slot) pairs
constexpr int kBlockCap = 16384;   // CTA bitonic sort in shared memory

__device__ __forceinline__ int axis_cell(double p, double c, double r, int K, double b,
                                         double y) {
    return exact_axis_cell(p, c, r, K, b, y);
}

__global__ void __launch_bounds__(256) k_keys(Geometry g, int64_t n, const double* __restrict__ xyz,
                                              int32_t* __restrict__ key, int32_t* __restrict__ rank,
                                              int32_t* __restrict__ cnt, unsigned long long* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p0 = xyz[3 * i], p1 = xyz[3 * i + 1], p2 = xyz[3 * i + 2];
    // Box3::contains (geometry.hpp:36-40)
    if (fabs(p0 - g.center[0]) > g.radius || fabs(p1 - g.center[1]) > g.radius ||
        fabs(p2 - g.center[2]) > g.radius)
        atomicMin(&bad[0], (unsigned long long)i);
    const double b = __dmul_rn(2.0, g.radius), y = g.inv_diam;
    const int c0 = axis_cell(p0, g.center[0], g.radius, g.K[0], b, y);
    const int c1 = axis_cell(p1, g.center[1], g.radius, g.K[1], b, y);
    const int c2 = axis_cell(p2, g.center[2], g.radius, g.K[2], b, y);
    if (c0 < g.x_lo || c0 >= g.x_hi || c1 < g.y_lo || c1 >= g.y_hi || c2 < g.z_lo || c2 >= g.z_hi)
        atomicOr(&bad[1], 2ull);  // not in this plan's cell block
    const int k = (c0 * g.K[1] + c1) * g.K[2] + c2;             // CellGrid::flatten
    key[i] = k;
    rank[i] = atomicAdd(&cnt[k], 1);  // provisional slot, fixed up by k_segsort
}

// Exclusive scan of the histogram by one CTA: chunks of kScanChunk counts,
// each warp scanning 512 consecutive counts 32 at a time with shuffles.
constexpr int kScanChunk = 16384;
__global__ void __launch_bounds__(1024) k_scan(int ncell, const int32_t* __restrict__ cnt,
                                               int32_t* __restrict__ start) {
    __shared__ int32_t wtot[32];
    __shared__ int32_t carry;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < ncell; base += kScanChunk) {
        int vals[16], own[16];
        int run = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int idx = base + w * 512 + k * 32 + lane;
            own[k] = idx < ncell ? cnt[idx] : 0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int v = own[k];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            vals[k] = run + v;  // inclusive within the warp's 512 counts
            run += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) wtot[w] = run;
        __syncthreads();
        if (w == 0) {
            int v = wtot[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            wtot[lane] = v;  // inclusive over warps
        }
        __syncthreads();
        const int off = carry + (w > 0 ? wtot[w - 1] : 0);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int idx = base + w * 512 + k * 32 + lane;
            if (idx < ncell) start[idx] = off + vals[k] - own[k];
        }
        __syncthreads();
        if (tid == 0) carry += wtot[31];
        __syncthreads();
    }
    if (tid == 0) start[ncell] = carry;
}

__global__ void __launch_bounds__(256) k_place(int64_t n, const int32_t* __restrict__ key,
                                               const int32_t* __restrict__ rank,
                                               const int32_t* __restrict__ start,
                                               int32_t* __restrict__ perm,
                                               const double* __restrict__ xyz,
                                               const double* __restrict__ q,
                                               double4* __restrict__ rec) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int pos = start[key[i]] + rank[i];
    perm[pos] = (int32_t)i;
    if (rec) rec[pos] = make_double4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], q[i]);
}

// move the record of provisional slot j (within the segment) to sorted slot r
__device__ __forceinline__ void move_rec(double4* sp, const double4* rec, int s0, int r, int j) {
    if (sp) sp[s0 + r] = rec[s0 + j];
}

// Warp rank sort of b[0..cnt) (distinct values, padded to P4 with INT_MAX):
// member k of lane l (provisional slot l + 32k) goes to slot
// (number of smaller members).
template <int V>
__device__ __forceinline__ void rank_sort(const int32_t* b, int P4, int cnt, int lane, int s0,
                                          int32_t* perm, double4* sp, const double4* rec) {
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
            perm[s0 + r[k]] = v[k];
            move_rec(sp, rec, s0, r[k], lane + 32 * k);
        }
}

// One warp per cell.
__global__ void __launch_bounds__(256) k_segsort_warp(int ncell, const int32_t* __restrict__ start,
                                                      int32_t* __restrict__ perm,
                                                      int32_t* __restrict__ big,
                                                      int32_t* __restrict__ nbig,
                                                      const double4* __restrict__ rec,
                                                      double4* __restrict__ sp) {
    __shared__ __align__(16) unsigned long long buf[8][kWarpCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * 8 + w;
    if (cell >= ncell) return;
    const int s0 = start[cell], cnt = start[cell + 1] - s0;
    if (cnt == 0) return;
    if (cnt == 1) {
        if (lane == 0) move_rec(sp, rec, s0, 0, 0);
        return;
    }
    if (cnt > kWarpCap) {
        if (lane == 0) big[atomicAdd(nbig, 1)] = cell;
        return;
    }
    if (cnt <= 32) {  // register bitonic network on (index, slot) pairs
        int v = lane < cnt ? perm[s0 + lane] : INT_MAX;
        int j = lane;
        for (int k = 2; k <= 32; k <<= 1)
            for (int d = k >> 1; d > 0; d >>= 1) {
                const int ov = __shfl_xor_sync(0xffffffffu, v, d);
                const int oj = __shfl_xor_sync(0xffffffffu, j, d);
                const bool up = (lane & k) == 0, lower = (lane & d) == 0;
                if ((lower == up) == (ov < v)) {
                    v = ov;
                    j = oj;
                }
            }
        if (lane < cnt) {
            perm[s0 + lane] = v;
            move_rec(sp, rec, s0, lane, j);
        }
        return;
    }
    if (cnt <= kRankCap) {
        int32_t* b = reinterpret_cast<int32_t*>(buf[w]);
        const int P4 = (cnt + 3) & ~3;
        for (int i = lane; i < P4; i += 32) b[i] = i < cnt ? perm[s0 + i] : INT_MAX;
        __syncwarp();
        if (cnt <= 128) rank_sort<4>(b, P4, cnt, lane, s0, perm, sp, rec);
        else rank_sort<8>(b, P4, cnt, lane, s0, perm, sp, rec);
        return;
    }
    // (index << 32 | slot) pairs, bitonic in shared memory
    unsigned long long* b = buf[w];
    int P = 512;
    while (P < cnt) P <<= 1;
    for (int i = lane; i < P; i += 32)
        b[i] = i < cnt ? ((unsigned long long)(unsigned)perm[s0 + i] << 32 | (unsigned)i) : ~0ull;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1)
        for (int d = k >> 1; d > 0; d >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixd = i ^ d;
                if (ixd > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long x = b[i], y = b[ixd];
                    if ((x > y) == up) {
                        b[i] = y;
                        b[ixd] = x;
                    }
                }
            }
            __syncwarp();
        }
    for (int i = lane; i < cnt; i += 32) {
        perm[s0 + i] = (int32_t)(b[i] >> 32);
        move_rec(sp, rec, s0, i, (int)(b[i] & 0xffffffffu));
    }
}

// Large cells: one CTA per cell. Up to kBlockCap members are sorted as
// (index, slot) pairs in shared memory; beyond that the CTA rebuilds the
// segment by a stable, in-order compaction over all keys (O(n) per huge
// cell, only for degenerate inputs) and gathers the records from the inputs.
__global__ void __launch_bounds__(1024) k_segsort_big(int64_t n, const int32_t* __restrict__ key,
                                                      const int32_t* __restrict__ start,
                                                      int32_t* __restrict__ perm,
                                                      const int32_t* __restrict__ big,
                                                      const int32_t* __restrict__ nbig,
                                                      const double4* __restrict__ rec,
                                                      double4* __restrict__ sp,
                                                      const double* __restrict__ xyz,
                                                      const double* __restrict__ q) {
    extern __shared__ unsigned long long sbuf[];
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
            for (int i = tid; i < P; i += T)
                sbuf[i] = i < cnt ? ((unsigned long long)(unsigned)perm[s0 + i] << 32 | (unsigned)i)
                                  : ~0ull;
            __syncthreads();
            for (int k = 2; k <= P; k <<= 1)
                for (int d = k >> 1; d > 0; d >>= 1) {
                    for (int i = tid; i < P; i += T) {
                        const int ixd = i ^ d;
                        if (ixd > i) {
                            const bool up = (i & k) == 0;
                            const unsigned long long x = sbuf[i], y = sbuf[ixd];
                            if ((x > y) == up) {
                                sbuf[i] = y;
                                sbuf[ixd] = x;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int i = tid; i < cnt; i += T) {
                perm[s0 + i] = (int32_t)(sbuf[i] >> 32);
                move_rec(sp, rec, s0, i, (int)(sbuf[i] & 0xffffffffu));
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
                if (hit) {
                    const int slot = s0 + before + __popc(m & ((1u << lane) - 1));
                    perm[slot] = (int32_t)i;
                    if (sp)
                        sp[slot] = make_double4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], q[i]);
                }
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

int blocks_for(int64_t n, int threads) { return (int)((n + threads - 1) / threads); }

}  // namespace

void launch_sort(const Geometry& g, int64_t n, const double* xyz, const SortBuffers& b,
                 cudaStream_t s, int* launches, const double* q, double4* sp) {
    if (!q) sp = nullptr;
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_segsort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBlockCap * (int)sizeof(unsigned long long)));
    });
    KB_CUDA(cudaMemsetAsync(b.cnt, 0, sizeof(int32_t) * g.ncell, s));
    KB_CUDA(cudaMemsetAsync(b.nbig, 0, sizeof(int32_t), s));
    if (n > 0) {
        k_keys<<<blocks_for(n, 256), 256, 0, s>>>(g, n, xyz, b.key, b.rank, b.cnt, b.bad);
        KB_CHECK_LAUNCH();
    }
    k_scan<<<1, 1024, 0, s>>>(g.ncell, b.cnt, b.start);
    KB_CHECK_LAUNCH();
    int l = 2;
    if (n > 0) {
        k_place<<<blocks_for(n, 256), 256, 0, s>>>(n, b.key, b.rank, b.start, b.perm, xyz, q,
                                                   sp ? b.rec : nullptr);
        KB_CHECK_LAUNCH();
        k_segsort_warp<<<(g.ncell + 7) / 8, 256, 0, s>>>(g.ncell, b.start, b.perm, b.big, b.nbig,
                                                         b.rec, sp);
        KB_CHECK_LAUNCH();
        k_segsort_big<<<sm_count(), 1024, kBlockCap * sizeof(unsigned long long), s>>>(
            n, b.key, b.start, b.perm, b.big, b.nbig, b.rec, sp, xyz, q);
        KB_CHECK_LAUNCH();
        l += 4;
    }
    if (launches) *launches += l;
}

void launch_permute(int64_t n, const double* xyz, const double* q, const int32_t* perm,
                    double4* sp, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t blk = (n + 255) / 256;
    k_permute<<<(int)(blk > sm_count() * 16 ? sm_count() * 16 : blk), 256, 0, s>>>(n, xyz, q, perm, sp);
    KB_CHECK_LAUNCH();
}

}  // namespace kb
