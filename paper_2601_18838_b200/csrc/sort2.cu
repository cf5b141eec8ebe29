// sort2.cu -- two-level stable counting sort into cell order (the default
// cell sort; sort.cu's atomic-slot sort is the fallback for very large grids).
//
// The reference's order (assign_particles, geometry.hpp:131-154) is: cells in
// flatten order (c0, c1, c2), particles ascending inside each cell. Here:
//   k_tile_hist   cell key (exact arithmetic, shared with sort.cu) and a
//                 per-tile histogram over columns (c0, c1)
//   k_col_scan    per column: exclusive scan over tiles, column totals
//   k_col_scatter stable scatter by column: inside a tile, ranks come from
//                 warp ballots in particle order plus per-warp offsets, so
//                 every column segment keeps ascending particle order; writes
//                 the packed (index, c2) pair and the particle record
//   k_z_sort      one CTA per column: stable counting sort by c2 in chunks
//                 staged in shared memory, so perm and the cell-ordered
//                 records leave in coalesced runs; writes cell_start
// No global atomics; the result is deterministic and equals the reference.
//
// Scattered global stores cost one L2 request per lane (measured:
// scripts/probes/scatter_probe.cu), so the design keeps them to one packed
// 8-byte pair plus one 32-byte record per particle (column scatter) and
// stages the per-column pass in shared memory.
#include <algorithm>
#include <climits>
#include <type_traits>

#include "internal.h"
#include "trace.h"

namespace kb {
namespace {

#ifndef SORT2_ROUNDS
#define SORT2_ROUNDS 8
#endif
#ifndef SORT2_ZROUNDS
#define SORT2_ZROUNDS 4
#endif
constexpr int kTileWarps = 8;
constexpr int kRounds = SORT2_ROUNDS;             // 32-particle rounds per warp
constexpr int kTile = kTileWarps * kRounds * 32;  // particles per tile (2048)
constexpr int kHistThreads = kTile / 4;           // 4 particles per thread
constexpr int kMinTile = 4 * 32 * kTileWarps;     // the smallest k_tile_sort tile (TR = 4)
constexpr int kGroup = 4;                         // rounds whose loads are issued together
constexpr int kZWarps = 8;                        // warps per column CTA in k_z_sort
constexpr int kZRounds = SORT2_ZROUNDS;
constexpr int kZChunk = kZWarps * kZRounds * 32;  // column elements staged per chunk
static_assert(kRounds % kGroup == 0, "rounds come in load groups");

// Markstein-division axis cell (internal.h):
__device__ __forceinline__ int axis_cell2(double p, double c, double r, int K, double b,
                                          double y) {
    return exact_axis_cell(p, c, r, K, b, y);
}

// Lanes of the warp holding the same non-negative key (inactive lanes pass a
// negative key and are never anyone's peer): one ballot per key bit, NB known
// at compile time (keys are < 2^NB). MATCH.ANY measured slower on B200.
// The votes are volatile asm so the compiler keeps them in program order:
// hoisting every round's ballots at once costs more registers than it saves.
__device__ __forceinline__ unsigned vote_ballot(bool p) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tvote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
        : "=r"(r)
        : "r"((unsigned)p));
    return r;
}

template <int NB>
__device__ __forceinline__ unsigned warp_peers(int v) {
    unsigned m = vote_ballot(v >= 0);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const bool bit = (v >> b) & 1;
        const unsigned bb = vote_ballot(bit);
        m &= bit ? bb : ~bb;
    }
    return m;
}

__host__ __device__ inline int bits_for(int count) {  // bits to hold 0..count-1
    int b = 0;
    while ((1 << b) < count) ++b;
    return b;
}

// Cell keys + box check + per-tile column histogram hist[col * ntiles + tile].
__global__ void __launch_bounds__(kHistThreads) k_tile_hist(Geometry g, int64_t n,
                                                   const double* __restrict__ xyz,
                                                   int32_t* __restrict__ key,
                                                   int32_t* __restrict__ hist, int ntiles,
                                                   unsigned long long* bad) {
    extern __shared__ int32_t h[];  // [ncol]
    const int ncol = g.K[0] * g.K[1];
    for (int c = threadIdx.x; c < ncol; c += blockDim.x) h[c] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    const double b = __dmul_rn(2.0, g.radius), y = g.inv_diam;
    constexpr int kPer = kTile / kHistThreads;
    double p[kPer][3];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {  // issue every load of the tile first
        const int64_t i = t0 + u * kHistThreads + threadIdx.x;
        if (i < n) {
            p[u][0] = __ldg(xyz + 3 * i);
            p[u][1] = __ldg(xyz + 3 * i + 1);
            p[u][2] = __ldg(xyz + 3 * i + 2);
        }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int64_t i = t0 + u * kHistThreads + threadIdx.x;
        if (i >= n) break;
        const double p0 = p[u][0], p1 = p[u][1], p2 = p[u][2];
        if (fabs(p0 - g.center[0]) > g.radius || fabs(p1 - g.center[1]) > g.radius ||
            fabs(p2 - g.center[2]) > g.radius)
            atomicMin(&bad[0], (unsigned long long)i);  // Box3::contains (geometry.hpp:36-40)
        const int c0 = axis_cell2(p0, g.center[0], g.radius, g.K[0], b, y);
        const int c1 = axis_cell2(p1, g.center[1], g.radius, g.K[1], b, y);
        const int c2 = axis_cell2(p2, g.center[2], g.radius, g.K[2], b, y);
        if (c0 < g.x_lo || c0 >= g.x_hi || c1 < g.y_lo || c1 >= g.y_hi || c2 < g.z_lo || c2 >= g.z_hi)
            atomicOr(&bad[1], 2ull);  // not in this plan's cell block
        key[i] = ((c0 * g.K[1] + c1) << 16) | c2;  // (column, c2) packed
        atomicAdd(&h[c0 * g.K[1] + c1], 1);  // shared-memory counter, order irrelevant
    }
    __syncthreads();
    for (int c = threadIdx.x; c < ncol; c += blockDim.x) hist[(int64_t)c * ntiles + blockIdx.x] = h[c];
}

// Exclusive scan of ctot[0..ncol) into out[0..ncol], out[ncol] = total; whole
// CTA (blockDim a multiple of 32, <= 1024); ends synchronised.
__device__ void block_col_bases(const int32_t* ctot, int ncol, int32_t* out,
                                int32_t* wsum /* [32] */) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nt = blockDim.x;
    const int per = (ncol + nt - 1) / nt;
    const int lo = min(ncol, tid * per), hi = min(ncol, lo + per);
    int s = 0;
    for (int c = lo; c < hi; ++c) s += ctot[c];
    int x = s;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = lane < (nt >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    int run = (w > 0 ? wsum[w - 1] : 0) + x - s;
    for (int c = lo; c < hi; ++c) {
        out[c] = run;
        run += ctot[c];
    }
    if (tid == nt - 1) out[ncol] = run;
    __syncthreads();
}

// Warp per column: exclusive scan of hist[col][0..ntiles) in place, column
// total to ctot[col]. Loads are issued kScanBatch x 32 at a time. The last CTA
// to finish (ticket counter, reset for the next launch) turns the totals into
// the column bases cbase[0..ncol] -- a fixed-order scan, so deterministic.
constexpr int kScanBatch = 8;
__global__ void __launch_bounds__(256) k_col_scan(int ncol, int ntiles, int32_t* __restrict__ hist,
                                                  int32_t* ctot, int32_t* cbase,
                                                  unsigned* ticket) {
    __shared__ int32_t wsum[32];
    __shared__ bool last;
    const int col = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (col < ncol) {
        int32_t* row = hist + (int64_t)col * ntiles;
        int carry = 0;
        for (int b0 = 0; b0 < ntiles; b0 += 32 * kScanBatch) {
            int v[kScanBatch];
#pragma unroll
            for (int u = 0; u < kScanBatch; ++u) {
                const int t = b0 + u * 32 + lane;
                v[u] = t < ntiles ? row[t] : 0;
            }
#pragma unroll
            for (int u = 0; u < kScanBatch; ++u) {
                int x = v[u];
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const int t = b0 + u * 32 + lane;
                if (t < ntiles) row[t] = carry + x - v[u];
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
        }
        if (lane == 0) ctot[col] = carry;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    block_col_bases(ctot, ncol, cbase, wsum);
    if (threadIdx.x == 0) *ticket = 0u;
}

// Stable scatter by column. Warp w of tile t owns particles
// [t*kTile + w*kRounds*32, +kRounds*32), processed 32 at a time in index order.
// The warp's keys are loaded into registers once and the record loads of
// kGroup rounds are issued together.
template <int CB>
__global__ void __launch_bounds__(kTileWarps * 32, 4) k_col_scatter(Geometry g, int64_t n, int ntiles,
                                                                 const int32_t* __restrict__ key,
                                                                 const int32_t* __restrict__ cscan,
                                                                 const int32_t* __restrict__ cbase,
                                                                 const double* __restrict__ xyz,
                                                                 const double* __restrict__ q,
                                                                 int32_t* __restrict__ idx2,
                                                                 double4* __restrict__ rec2) {
    // [kTileWarps][ncol] per-warp column counters, then offsets inside the
    // tile's column segment (16-bit: a tile holds kTile particles), and the
    // tile's global column bases [ncol] (half the shared memory of 32-bit
    // counters: a fourth CTA per SM on large grids)
    extern __shared__ int32_t csm[];
    uint16_t* wc = reinterpret_cast<uint16_t*>(csm);
    __shared__ unsigned pm[kTileWarps][kRounds][32];  // phase-1 peer masks, reused in phase 3
    const int ncol = g.K[0] * g.K[1];
    int32_t* cbs = csm + (kTileWarps * ncol + 1) / 2;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < kTileWarps * ncol; e += blockDim.x) wc[e] = 0;
    const int64_t wbase = (int64_t)blockIdx.x * kTile + w * (kRounds * 32);
    int kreg[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        kreg[r] = i < n ? __ldg(key + i) : -1;
    }
    __syncthreads();
    // 1: per-warp column counts
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const bool act = kreg[r] >= 0;
        const int col = act ? kreg[r] >> 16 : -1 - lane;
        const unsigned peers = warp_peers<CB>(col);
        pm[w][r][lane] = peers;
        if (act && lane == __ffs(peers) - 1) wc[w * ncol + col] += (uint16_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // 2: exclusive prefix over warps; this tile's global column offset
    for (int c = threadIdx.x; c < ncol; c += blockDim.x) {
        cbs[c] = cbase[c] + cscan[(int64_t)c * ntiles + blockIdx.x];
        int run = 0;
        for (int k = 0; k < kTileWarps; ++k) {
            const int t = wc[k * ncol + c];
            wc[k * ncol + c] = (uint16_t)run;
            run += t;
        }
    }
    __syncthreads();
    // 3: placement in index order, one load group at a time (keys re-read
    // from L1/L2): ranks first, then the record loads, then the stores
#pragma unroll 1
    for (int r0 = 0; r0 < kRounds; r0 += kGroup) {
        int kg[kGroup], pos[kGroup];
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
            const int64_t i = wbase + (r0 + u) * 32 + lane;
            kg[u] = i < n ? __ldg(key + i) : -1;
        }
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
            const int k = kg[u];
            const bool act = k >= 0;
            const int col = act ? k >> 16 : -1 - lane;
            const unsigned peers = pm[w][r0 + u][lane];
            int rel = 0, base = 0;
            if (act) {
                rel = wc[w * ncol + col];
                base = cbs[col];
            }
            pos[u] = base + rel + __popc(peers & ((1u << lane) - 1));
            __syncwarp();
            if (act && lane == __ffs(peers) - 1) wc[w * ncol + col] = (uint16_t)(rel + __popc(peers));
            __syncwarp();
        }
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
            const int k = kg[u];
            if (k < 0) continue;
            const int64_t i = wbase + (r0 + u) * 32 + lane;
            idx2[pos[u]] = (int32_t)i;
            st_rec(rec2 + pos[u], make_double4(__ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1),
                                               __ldg(xyz + 3 * i + 2), q ? __ldg(q + i) : 0.0));
        }
    }
}

// Bulk (TMA) global -> shared copies completing on an mbarrier.
#ifdef ZSORT_PROFILE
__device__ __forceinline__ unsigned __smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// bytes is a multiple of 16; pieces of at most 32 KB
__device__ __forceinline__ void bulk_g2s_pieces(void* dst, const void* src, unsigned bytes,
                                                uint64_t* bar) {
    for (unsigned o = 0; o < bytes; o += 32768u)
        bulk_g2s(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                 min(32768u, bytes - o), bar);
}

// c2 of a staged particle record: the same exact arithmetic as the key.
__device__ __forceinline__ int rec_c2(const Geometry& g, const double4& r) {
    return axis_cell2(r.z, g.center[2], g.radius, g.K[2], __dmul_rn(2.0, g.radius), g.inv_diam);
}

// Whole-column variant: a column of up to kZCap particles is staged in shared
// memory in one go (records and indices, by bulk copies), ranked with
// per-thread counters (thread t owns a contiguous slice of the column; the
// [c2][thread] counters are scanned in that order, which is exactly stable
// order) and written out in cell order as one contiguous run.
constexpr int kZCap = 2560;  // <= 10 particles per thread (4-bit counters)
constexpr int kZThreads = kZWarps * 32;
struct ZWholeLayout {
    size_t rec, idx, inv, z, cnt, total;
    __host__ __device__ ZWholeLayout(int K2, int cap) {
        rec = 0;
        idx = sizeof(double4) * cap;
        inv = idx + sizeof(int32_t) * (cap + 4);
        z = inv + sizeof(uint16_t) * cap;
        cnt = z + sizeof(uint8_t) * cap;
        cnt = (cnt + 15) & ~size_t(15);
        total = cnt + sizeof(uint16_t) * (size_t)K2 * kZThreads;
    }
};
constexpr size_t kZWholeMaxSmem = 112 * 1024;  // two CTAs per SM
// Largest whole-column capacity whose layout keeps two CTAs per SM (the z
// counters grow with K2: config 4's 43 cells per column fit 2048); 0: none.
__host__ inline int whole_cap_for(int K2) {
    if (K2 > 64) return 0;
    for (int cap = kZCap; cap >= 1024; cap -= 512)
        if (ZWholeLayout(K2, cap).total <= kZWholeMaxSmem) return cap;
    return 0;
}

// Steps 2-5 of the whole-column sort: the column's m records and indices are
// staged in shared memory in ascending particle order and cnt is zeroed.
template <int ZB, class ZOf, class Emit>
__device__ __forceinline__ void z_whole_core(const Geometry& g, int col, int cs, int m, int64_t n,
                                             ZOf zof, Emit emit, uint16_t* s_inv, uint8_t* s_z,
                                             uint16_t* cnt, int32_t* __restrict__ start,
                                             int32_t* wsum) {
    const int K2 = g.K[2], ncol = g.K[0] * g.K[1];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#ifdef ZSORT_PROFILE
    long long T[8];
    int nT = 0;
    T[nT++] = clock64();
#define ZSTAMP() T[nT++] = clock64()
#else
#define ZSTAMP()
#endif
    // 2: per-thread counts over the thread's contiguous slice, kept as 4-bit
    // counters packed in registers (at most 10 particles per thread)
    // four named 64-bit words of 16 counters (c2 < 64); named, not an
    // array, so they stay in registers
    static_assert(ZB <= 6, "whole-column path handles up to 64 cells per column");
    const int per = (m + kZThreads - 1) / kZThreads;
    const int lo = min(m, tid * per), hi = min(m, lo + per);
    unsigned long long n0 = 0, n1 = 0, n2 = 0, n3 = 0;
    for (int j = lo; j < hi; ++j) {
        const int z = zof(j);
        s_z[j] = (uint8_t)z;
        const unsigned long long inc = 1ull << ((z & 15) * 4);
        const int wq = z >> 4;
        n0 += wq == 0 ? inc : 0ull;
        n1 += wq == 1 ? inc : 0ull;
        n2 += wq == 2 ? inc : 0ull;
        n3 += wq == 3 ? inc : 0ull;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r < K2) cnt[r * kZThreads + tid] = (uint16_t)((n0 >> (4 * r)) & 15u);
        if (16 + r < K2) cnt[(16 + r) * kZThreads + tid] = (uint16_t)((n1 >> (4 * r)) & 15u);
        if (32 + r < K2) cnt[(32 + r) * kZThreads + tid] = (uint16_t)((n2 >> (4 * r)) & 15u);
        if (48 + r < K2) cnt[(48 + r) * kZThreads + tid] = (uint16_t)((n3 >> (4 * r)) & 15u);
    }
    __syncthreads();
    ZSTAMP();
    TRACE_MARK(1, 3);
    // 3: exclusive scan of the counters in (c2, thread) order: thread t scans
    // the K2 consecutive entries [t*K2, (t+1)*K2)
    {
        uint16_t* strip = cnt + tid * K2;
        int sum = 0;
        for (int i = 0; i < K2; ++i) sum += strip[i];
        int x = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        int off = 0;
        for (int k = 0; k < w; ++k) off += wsum[k];
        int run = off + x - sum;
        for (int i = 0; i < K2; ++i) {
            const int t = strip[i];
            strip[i] = (uint16_t)run;
            run += t;
        }
    }
    __syncthreads();
    ZSTAMP();
    TRACE_MARK(1, 4);
    for (int z = tid; z < K2; z += kZThreads) start[(int64_t)col * K2 + z] = cs + cnt[z * kZThreads];
    if (col == ncol - 1 && tid == 0) start[(int64_t)ncol * K2] = (int)n;
    // 4: stable ranks -> inverse permutation (running 4-bit counters again)
    n0 = n1 = n2 = n3 = 0;
    for (int j = lo; j < hi; ++j) {
        const int z = s_z[j];
        const int sh = (z & 15) * 4, wq = z >> 4;
        const unsigned long long cur = wq == 0 ? n0 : wq == 1 ? n1 : wq == 2 ? n2 : n3;
        const int off = (int)((cur >> sh) & 15u);
        const unsigned long long inc = 1ull << sh;
        n0 += wq == 0 ? inc : 0ull;
        n1 += wq == 1 ? inc : 0ull;
        n2 += wq == 2 ? inc : 0ull;
        n3 += wq == 3 ? inc : 0ull;
        s_inv[cnt[z * kZThreads + tid] + off] = (uint16_t)j;
    }
    __syncthreads();
    ZSTAMP();
    TRACE_MARK(1, 5);
    // 5: the column leaves in cell order as one contiguous run
    emit(s_inv);
#ifdef ZSORT_PROFILE
    __syncthreads();
    ZSTAMP();
    if (tid == 0 && (col % 37 == 0))
        printf("zsort col %d sm %d m %d: load %lld count %lld scan %lld rank %lld write %lld start %lld\n", col,
               (int)__smid(), m, T[1] - T[0], T[2] - T[1], T[3] - T[2], T[4] - T[3], T[5] - T[4], T[0]);
#endif
#undef ZSTAMP
}

// The record path: c2 recomputed from the staged record, records written out.
template <int ZB>
__device__ __forceinline__ void z_whole_body(const Geometry& g, int col, int cs, int m, int64_t n,
                                             const double4* s_rec, const int32_t* s_idx,
                                             uint16_t* s_inv, uint8_t* s_z, uint16_t* cnt,
                                             int32_t* __restrict__ perm, int32_t* __restrict__ start,
                                             double4* __restrict__ sp, int32_t* wsum) {
    z_whole_core<ZB>(
        g, col, cs, m, n, [&](int j) { return rec_c2(g, s_rec[j]); },
        [&](const uint16_t* inv) {
            for (int k = threadIdx.x; k < m; k += kZThreads) {
                const int j = inv[k];
                perm[cs + k] = s_idx[j];
                if (sp) st_rec(sp + cs + k, s_rec[j]);
            }
        },
        s_inv, s_z, cnt, start, wsum);
}

// Record i from the input arrays with two loads for (x, y, z): the 24-byte
// triple is either 16-byte aligned ((x, y) as one 128-bit load, then z) or 8
// bytes past ((y, z) as the 128-bit load after x), decided on the address. A scattered warp load costs one
// L1 wavefront per lane, so this is 3 instead of 4 per record with q.
__device__ __forceinline__ double4 gather_rec(const double* __restrict__ xyz, const double* __restrict__ q,
                                              int64_t i) {
    const double* base = xyz + 3 * i;
#ifdef REC_LD4  // A/B: three 8-byte loads for (x, y, z)
    return make_double4(__ldg(base), __ldg(base + 1), __ldg(base + 2), q ? __ldg(q + i) : 0.0);
#else
    const int odd = (int)((reinterpret_cast<uintptr_t>(base) >> 3) & 1);
    const double2 v = __ldg(reinterpret_cast<const double2*>(base + odd));
    const double s = __ldg(base + (odd ? 0 : 2));
    return make_double4(odd ? s : v.x, odd ? v.x : v.y, odd ? v.y : s, q ? __ldg(q + i) : 0.0);
#endif
}
// The key path (k_z_tiles_ko): staged (particle, c2) pairs; the records are
// gathered from the input arrays (L2-resident after the tile pass) straight
// into their sorted place, four at a time per thread.
template <int ZB>
__device__ __forceinline__ void z_whole_pairs(const Geometry& g, int col, int cs, int m, int64_t n,
                                              const int2* s_pair, uint16_t* s_inv, uint8_t* s_z,
                                              uint16_t* cnt, int32_t* __restrict__ perm,
                                              int32_t* __restrict__ start, const double* __restrict__ xyz,
                                              const double* __restrict__ q, double4* __restrict__ sp,
                                              int32_t* wsum) {
    z_whole_core<ZB>(
        g, col, cs, m, n, [&](int j) { return s_pair[j].y; },
        [&](const uint16_t* inv) {
            for (int k0 = threadIdx.x; k0 < m; k0 += 4 * kZThreads) {
                int id[4];
                double4 r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = k0 + u * kZThreads;
                    id[u] = k < m ? s_pair[inv[k]].x : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (sp && id[u] >= 0) r[u] = gather_rec(xyz, q, id[u]);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (id[u] >= 0) {
                        const int k = k0 + u * kZThreads;
                        perm[cs + k] = id[u];
                        if (sp) st_rec(sp + cs + k, r[u]);
                    }
            }
        },
        s_inv, s_z, cnt, start, wsum);
}

template <int ZB>
__device__ __forceinline__ void z_sort_whole(const Geometry& g, int col, int cs, int m,
                                             int64_t n, const int32_t* __restrict__ idx2,
                                             const double4* __restrict__ rec2,
                                             int32_t* __restrict__ perm,
                                             int32_t* __restrict__ start,
                                             double4* __restrict__ sp, unsigned char* zsm,
                                             uint64_t* bar, int32_t* wsum, int cap) {
    const int K2 = g.K[2];
    const ZWholeLayout L(K2, cap);
    double4* s_rec = reinterpret_cast<double4*>(zsm + L.rec);
    int32_t* s_idx = reinterpret_cast<int32_t*>(zsm + L.idx);
    uint16_t* s_inv = reinterpret_cast<uint16_t*>(zsm + L.inv);
    uint8_t* s_z = reinterpret_cast<uint8_t*>(zsm + L.z);
    uint16_t* cnt = reinterpret_cast<uint16_t*>(zsm + L.cnt);  // [K2][kZThreads]
    const int tid = threadIdx.x;
    // 1: stage the column with bulk copies (indices from the multiple of 4 at
    // or below cs, so both ends are 16-byte aligned; idx2 has 4 spare slots)
    const int cs_al = cs & ~3, m_al = ((cs + m + 3) & ~3) - cs_al;
    if (tid == 0) {
        mbar_init(bar, 1);
        const unsigned brec = 32u * (unsigned)m, bidx = 4u * (unsigned)m_al;
        mbar_expect_tx(bar, brec + bidx);
        if (brec) bulk_g2s_pieces(s_rec, rec2 + cs, brec, bar);
        if (bidx) bulk_g2s_pieces(s_idx, idx2 + cs_al, bidx, bar);
    }
    for (int e = tid; e < K2 * kZThreads; e += kZThreads) cnt[e] = 0;
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(bar, 0);
    s_idx += cs - cs_al;
    z_whole_body<ZB>(g, col, cs, m, n, s_rec, s_idx, s_inv, s_z, cnt, perm, start, sp, wsum);
}

// Chunked fallback for columns above kZCap (or grids whose counters do not
// fit): the segment is taken kZChunk elements at a time (warp w owns a
// contiguous kZRounds x 32 slice of the chunk); each chunk is ranked into
// shared memory in (c2, particle) order and written out as contiguous
// per-cell runs.
struct ZLayout {
    size_t rec, idx, z, cnt, zrun, lstart, total;
    __host__ __device__ explicit ZLayout(int K2) {
        rec = 0;
        idx = sizeof(double4) * kZChunk;
        z = idx + sizeof(int32_t) * kZChunk;
        cnt = z + sizeof(uint16_t) * kZChunk;
        cnt = (cnt + 15) & ~size_t(15);
        zrun = cnt + sizeof(int32_t) * kZWarps * K2;
        lstart = zrun + sizeof(int32_t) * K2;
        total = lstart + sizeof(int32_t) * (K2 + 1);
    }
};

// src(j) is the position in rec2/idx2 of the column's j-th particle in
// ascending particle order.
struct ContiguousSrc {
    int cs;
    __device__ int64_t operator()(int j) const { return (int64_t)cs + j; }
};
// Element access of the chunked column sort: records (rec2, idx2) or the key
// path's (particle, c2) pairs with the records gathered from the inputs.
struct RecAcc {
    const Geometry* g;
    const int32_t* idx2;
    const double4* rec2;
    __device__ int z(int64_t sj) const { return rec_c2(*g, ld_rec(rec2 + sj)); }
    __device__ int idx(int64_t sj) const { return __ldg(idx2 + sj); }
    __device__ double4 rec(int64_t sj, int) const { return ld_rec(rec2 + sj); }
};
struct PairAcc {
    const int2* pairs;
    const double* xyz;
    const double* q;
    __device__ int z(int64_t sj) const { return __ldg(&pairs[sj].y); }
    __device__ int idx(int64_t sj) const { return __ldg(&pairs[sj].x); }
    __device__ double4 rec(int64_t, int i) const { return gather_rec(xyz, q, i); }
};
template <int ZB, class Src, class Acc>
__device__ __forceinline__ void z_sort_chunked_acc(const Geometry& g, int col, int cs, int m, Src src,
                                                   Acc acc, int64_t n, int32_t* __restrict__ perm,
                                                   int32_t* __restrict__ start,
                                                   double4* __restrict__ sp, unsigned char* zsm);
template <int ZB, class Src>
__device__ __forceinline__ void z_sort_chunked(const Geometry& g, int col, int cs, int m, Src src,
                                               int64_t n, const int32_t* __restrict__ idx2,
                                               const double4* __restrict__ rec2,
                                               int32_t* __restrict__ perm,
                                               int32_t* __restrict__ start,
                                               double4* __restrict__ sp, unsigned char* zsm) {
    z_sort_chunked_acc<ZB>(g, col, cs, m, src, RecAcc{&g, idx2, rec2}, n, perm, start, sp, zsm);
}
template <int ZB, class Src, class Acc>
__device__ __forceinline__ void z_sort_chunked_acc(const Geometry& g, int col, int cs, int m, Src src,
                                                   Acc acc, int64_t n, int32_t* __restrict__ perm,
                                                   int32_t* __restrict__ start,
                                                   double4* __restrict__ sp, unsigned char* zsm) {
    const int K2 = g.K[2], ncol = g.K[0] * g.K[1];
    const ZLayout L(K2);
    double4* s_rec = reinterpret_cast<double4*>(zsm + L.rec);
    int32_t* s_idx = reinterpret_cast<int32_t*>(zsm + L.idx);
    uint16_t* s_z = reinterpret_cast<uint16_t*>(zsm + L.z);
    int32_t* cnt = reinterpret_cast<int32_t*>(zsm + L.cnt);  // [K2][kZWarps]
    int32_t* zrun = reinterpret_cast<int32_t*>(zsm + L.zrun);
    int32_t* lstart = reinterpret_cast<int32_t*>(zsm + L.lstart);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int e = tid; e < K2; e += kZThreads) zrun[e] = 0;
    __syncthreads();
    // column histogram over c2 (order-free)
    for (int j = tid; j < m; j += kZThreads) atomicAdd(&zrun[acc.z(src(j))], 1);
    __syncthreads();
    if (w == 0) {  // cell starts; zrun becomes each cell's running output position
        int carry = cs;
        for (int base = 0; base < K2; base += 32) {
            const int z = base + lane;
            const int own = z < K2 ? zrun[z] : 0;
            int x = own;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (z < K2) {
                zrun[z] = carry + x - own;
                start[(int64_t)col * K2 + z] = carry + x - own;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (col == ncol - 1 && lane == 0) start[(int64_t)ncol * K2] = (int)n;
    }
    for (int c0 = 0; c0 < m; c0 += kZChunk) {
        const int cm = min(kZChunk, m - c0);
        for (int e = tid; e < kZWarps * K2; e += kZThreads) cnt[e] = 0;
        int zr[kZRounds], ir[kZRounds];
        double4 v[kZRounds];
#pragma unroll
        for (int u = 0; u < kZRounds; ++u) {
            const int jl = w * (kZRounds * 32) + u * 32 + lane;
            zr[u] = -1 - lane;
            if (jl < cm) {
                const int64_t sj = src(c0 + jl);
                ir[u] = acc.idx(sj);
                zr[u] = acc.z(sj);
                if (sp) v[u] = acc.rec(sj, ir[u]);
            }
        }
        __syncthreads();
        unsigned pk[kZRounds];
#pragma unroll
        for (int u = 0; u < kZRounds; ++u) {
            const unsigned peers = warp_peers<ZB>(zr[u]);
            pk[u] = peers;
            if (zr[u] >= 0 && lane == __ffs(peers) - 1) cnt[zr[u] * kZWarps + w] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        if (w == 0) {  // exclusive offsets in (c2, warp) order; chunk-local cell starts
            int carry = 0;
            for (int z0 = 0; z0 < K2; z0 += 32) {
                const int z = z0 + lane;
                int own = 0;
                if (z < K2) {
#pragma unroll
                    for (int k = 0; k < kZWarps; ++k) {
                        const int t = cnt[z * kZWarps + k];
                        cnt[z * kZWarps + k] = own;
                        own += t;
                    }
                }
                int x = own;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (z < K2) {
                    const int ex = carry + x - own;
                    lstart[z] = ex;
#pragma unroll
                    for (int k = 0; k < kZWarps; ++k) cnt[z * kZWarps + k] += ex;
                }
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) lstart[K2] = carry;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kZRounds; ++u) {
            const bool act = zr[u] >= 0;
            const unsigned peers = pk[u];
            int base = 0;
            if (act) {
                base = cnt[zr[u] * kZWarps + w];
                const int lp = base + __popc(peers & ((1u << lane) - 1));
                s_idx[lp] = ir[u];
                s_z[lp] = (uint16_t)zr[u];
                if (sp) s_rec[lp] = v[u];
            }
            __syncwarp();
            if (act && lane == __ffs(peers) - 1) cnt[zr[u] * kZWarps + w] = base + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        for (int k = tid; k < cm; k += kZThreads) {  // contiguous per-cell runs
            const int z = s_z[k];
            const int gp = zrun[z] + (k - lstart[z]);
            perm[gp] = s_idx[k];
            if (sp) st_rec(sp + gp, s_rec[k]);
        }
        __syncthreads();
        for (int z = tid; z < K2; z += kZThreads) zrun[z] += lstart[z + 1] - lstart[z];
    }
}

// One CTA per column: stable counting sort of the column segment by c2.
template <int ZB>
__global__ void __launch_bounds__(kZThreads, 2) k_z_sort(Geometry g,
                                                       const int32_t* __restrict__ cbase,
                                                       int64_t n, int whole_cap,
                                                       const int32_t* __restrict__ idx2,
                                                       const double4* __restrict__ rec2,
                                                       int32_t* __restrict__ perm,
                                                       int32_t* __restrict__ start,
                                                       double4* __restrict__ sp) {
    extern __shared__ __align__(16) unsigned char zsm[];
    __shared__ int32_t wsum[32];
    __shared__ uint64_t zbar;
    const int col = blockIdx.x;
    const int cs = __ldg(cbase + col), m = __ldg(cbase + col + 1) - cs;
    if (ZB <= 6 && m <= whole_cap)  // uniform per CTA
        z_sort_whole<(ZB <= 6 ? ZB : 6)>(g, col, cs, m, n, idx2, rec2, perm, start, sp, zsm, &zbar, wsum,
                                         whole_cap);
    else
        z_sort_chunked<ZB>(g, col, cs, m, ContiguousSrc{cs}, n, idx2, rec2, perm, start, sp, zsm);
}

// ---- tile-sorted variant (the default where it fits) ----------------------
// k_tile_sort   one CTA per tile of kTile particles: cell keys, box checks and a
//               stable tile-local counting sort by column in shared memory; the
//               tile leaves column-ordered as one contiguous run, with its
//               column offsets toff[tile][0..ncol]
// k_z_tiles     one CTA per column: the column's piece of every tile gathered
//               in ascending tile order (= ascending particle order), then the
//               whole-column z sort above. Its base is sum_t toff[t][col]: a
//               tile's offset of the column counts exactly the tile's particles
//               of the earlier columns.
// This replaces k_tile_hist + k_col_scan + k_col_scatter: no cross-tile scan,
// and no scattered 32-byte record stores (scripts/probes/scatter_probe.cu).
struct TileLayout {
    size_t rec, idx, wc, tc, cb, total;
    __host__ __device__ TileLayout(int ncol, int tile) {
        rec = 0;
        idx = rec + sizeof(double4) * tile;
        wc = idx + sizeof(int32_t) * tile;
        tc = wc + ((sizeof(uint16_t) * kTileWarps * ncol + 15) & ~size_t(15));
        cb = tc + sizeof(int32_t) * ncol;
        total = cb + sizeof(int32_t) * (ncol + 1);
    }
};
constexpr size_t kTileMaxSmem = 200 * 1024;

// TR rounds of 32 particles per warp: tiles of TR * 256 particles (the host
// picks TR per launch to even out the last wave, launch_sort2_tiles).
template <int CB, int TR>
__global__ void __launch_bounds__(kTileWarps * 32, 2) k_tile_sort(Geometry g, int64_t n,
                                                               const double* __restrict__ xyz,
                                                               const double* __restrict__ q,
                                                               int32_t* __restrict__ toff,
                                                               int32_t* __restrict__ idx2,
                                                               double4* __restrict__ rec2,
                                                               unsigned long long* bad) {
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ int32_t wsum[32];
    const int ncol = g.K[0] * g.K[1];
    constexpr int kTT = TR * 32 * kTileWarps;
    const TileLayout TL(ncol, kTT);
    double4* s_rec = reinterpret_cast<double4*>(tsm + TL.rec);
    int32_t* s_idx = reinterpret_cast<int32_t*>(tsm + TL.idx);
    uint16_t* wc = reinterpret_cast<uint16_t*>(tsm + TL.wc);  // [kTileWarps][ncol]
    int32_t* tc = reinterpret_cast<int32_t*>(tsm + TL.tc);    // [ncol] tile column counts
    int32_t* cb = reinterpret_cast<int32_t*>(tsm + TL.cb);    // [ncol + 1] tile column starts
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int e = tid; e < (int)((TL.tc - TL.wc) / 16); e += blockDim.x)
        reinterpret_cast<uint4*>(wc)[e] = make_uint4(0u, 0u, 0u, 0u);
    const int64_t tbase = (int64_t)blockIdx.x * kTT;
    const int64_t wbase = tbase + w * (TR * 32);
    double4 rv[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {  // every load of the warp's slice in flight
        const int64_t i = wbase + r * 32 + lane;
        if (i < n)
            rv[r] = make_double4(__ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2),
                                 q ? __ldg(q + i) : 0.0);
    }
    const double b = __dmul_rn(2.0, g.radius), y = g.inv_diam;
    const bool zblock = g.z_lo > 0 || g.z_hi < g.K[2];
    int colr[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        colr[r] = -1;
        if (i < n) {
            const double p0 = rv[r].x, p1 = rv[r].y, p2 = rv[r].z;
            if (fabs(p0 - g.center[0]) > g.radius || fabs(p1 - g.center[1]) > g.radius ||
                fabs(p2 - g.center[2]) > g.radius)
                atomicMin(&bad[0], (unsigned long long)i);  // Box3::contains (geometry.hpp:36-40)
            const int c0 = axis_cell2(p0, g.center[0], g.radius, g.K[0], b, y);
            const int c1 = axis_cell2(p1, g.center[1], g.radius, g.K[1], b, y);
            // c2 only for plans with a z block (a clamped c2 is always in [0, K2))
            const int c2 = zblock ? axis_cell2(p2, g.center[2], g.radius, g.K[2], b, y) : g.z_lo;
            if (c0 < g.x_lo || c0 >= g.x_hi || c1 < g.y_lo || c1 >= g.y_hi || c2 < g.z_lo || c2 >= g.z_hi)
                atomicOr(&bad[1], 2ull);  // not in this plan's cell block
            colr[r] = c0 * g.K[1] + c1;
        }
    }
    __syncthreads();
    // 1: per-warp column counts (peer masks kept for the placement)
    unsigned pk[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const bool act = colr[r] >= 0;
        const int col = act ? colr[r] : -1 - lane;
        const unsigned peers = warp_peers<CB>(col);
        pk[r] = peers;
        if (act && lane == __ffs(peers) - 1) wc[w * ncol + col] += (uint16_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // 2: exclusive over warps inside each column, column totals, then the
    // exclusive scan over columns: the tile's column-ordered layout
    for (int c = tid; c < ncol; c += blockDim.x) {
        int run = 0;
#pragma unroll
        for (int k = 0; k < kTileWarps; ++k) {
            const int t = wc[k * ncol + c];
            wc[k * ncol + c] = (uint16_t)run;
            run += t;
        }
        tc[c] = run;
    }
    __syncthreads();
    block_col_bases(tc, ncol, cb, wsum);
    int32_t* trow = toff + (int64_t)blockIdx.x * (ncol + 1);
    for (int c = tid; c <= ncol; c += blockDim.x) trow[c] = cb[c];
    // 3: placement in index order into the staged tile
#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const bool act = colr[r] >= 0;
        const unsigned peers = pk[r];
        int base = 0;
        if (act) base = cb[colr[r]] + wc[w * ncol + colr[r]];
        __syncwarp();
        if (act) {
            if (lane == __ffs(peers) - 1) wc[w * ncol + colr[r]] += (uint16_t)__popc(peers);
            const int pos = base + __popc(peers & ((1u << lane) - 1));
            s_rec[pos] = rv[r];
            s_idx[pos] = (int32_t)(wbase + r * 32 + lane);
        }
        __syncwarp();
    }
    __syncthreads();
    // 4: the tile leaves as one contiguous run
    const int tn = cb[ncol];
    for (int k = tid; k < tn; k += blockDim.x) {
        st_rec(rec2 + tbase + k, s_rec[k]);
        idx2[tbase + k] = s_idx[k];
    }
}

__device__ __forceinline__ void cp_async16_s(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4_s(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// The column's piece tables: pre[t] = column-local start of tile t's piece
// (pre[ntiles] = m), srca[t] = the piece's position in rec2/idx2.
struct PieceSrc {
    const int32_t* pre;
    const int32_t* srca;
    int ntiles;
    __device__ int64_t operator()(int j) const {
        int lo = 0, hi = ntiles;  // largest t with pre[t] <= j
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= j) lo = mid; else hi = mid;
        }
        return (int64_t)srca[lo] + (j - pre[lo]);
    }
};

// Shared-memory plan of k_z_tiles (host and device agree on it).
struct ZTilesLayout {
    size_t tables, total_whole, total_chunked;
    __host__ __device__ ZTilesLayout(int K2, int ntiles, int cap) {
        const size_t tb = sizeof(int32_t) * (2 * (size_t)ntiles + 1);
        // the whole path needs no tables (each thread stages its own pieces)
        total_whole = cap > 0 ? ZWholeLayout(K2, cap).total : 0;
        tables = ZLayout(K2).total;  // chunked path
        total_chunked = tables + tb;
    }
};

template <int ZB>
__global__ void __launch_bounds__(kZThreads, 2) k_z_tiles(Geometry g, int64_t n, int ntiles, int tile,
                                                        int whole_cap,
                                                        const int32_t* __restrict__ toff,
                                                        const int32_t* __restrict__ idx2,
                                                        const double4* __restrict__ rec2,
                                                        int32_t* __restrict__ perm,
                                                        int32_t* __restrict__ start,
                                                        double4* __restrict__ sp) {
    extern __shared__ __align__(16) unsigned char zsm[];
    __shared__ int32_t wsum[32];
    const int col = blockIdx.x, ncol = g.K[0] * g.K[1], K2 = g.K[2];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    // every tile's piece of this column: thread-contiguous slices of tiles, so
    // the scan below is in tile order; the column base cs sums the pieces'
    // offsets and m their lengths
    const int per = (ntiles + kZThreads - 1) / kZThreads;
    const int lo = min(ntiles, tid * per), hi = min(ntiles, lo + per);
    const ZTilesLayout TL(K2, ntiles, whole_cap);
    int a_[4], e_[4];
    int csum = 0, psum = 0;
    if (per <= 4) {  // loads in flight together (every shape the tile path takes)
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lo + u < hi) {
                a_[u] = __ldg(toff + (int64_t)(lo + u) * (ncol + 1) + col);
                e_[u] = __ldg(toff + (int64_t)(lo + u) * (ncol + 1) + col + 1);
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lo + u < hi) {
                csum += a_[u];
                psum += e_[u] - a_[u];
            }
    } else {
        for (int t = lo; t < hi; ++t) {
            const int a = __ldg(toff + (int64_t)t * (ncol + 1) + col);
            csum += a;
            psum += __ldg(toff + (int64_t)t * (ncol + 1) + col + 1) - a;
        }
    }
    int x = psum, cx = csum;
    for (int o = 1; o < 32; o <<= 1) {
        const int y1 = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y1;
        cx += __shfl_xor_sync(0xffffffffu, cx, o);
    }
    if (lane == 31) wsum[w] = x;
    if (lane == 0) wsum[16 + w] = cx;
    __syncthreads();
    int off = 0, cs = 0;
    for (int k = 0; k < kZWarps; ++k) {
        off += k < w ? wsum[k] : 0;
        cs += wsum[16 + k];
    }
    int m = 0;
    for (int k = 0; k < kZWarps; ++k) m += wsum[k];
    const bool whole = ZB <= 6 && m <= whole_cap;  // uniform per CTA
    int run = off + x - psum;
    if (!whole) {  // piece tables past the chunked layout, binary-searched per element
        int32_t* pre = reinterpret_cast<int32_t*>(zsm + TL.tables);
        int32_t* srca = pre + ntiles + 1;
        for (int t = lo; t < hi; ++t) {
            const int a = __ldg(toff + (int64_t)t * (ncol + 1) + col);
            srca[t] = t * tile + a;
            pre[t] = run;
            run += __ldg(toff + (int64_t)t * (ncol + 1) + col + 1) - a;
        }
        if (tid == 0) pre[ntiles] = m;
        __syncthreads();
        z_sort_chunked<ZB>(g, col, cs, m, PieceSrc{pre, srca, ntiles}, n, idx2, rec2, perm, start, sp,
                           zsm);
        return;
    }
    const ZWholeLayout L(K2, whole_cap);
    double4* s_rec = reinterpret_cast<double4*>(zsm + L.rec);
    int32_t* s_idx = reinterpret_cast<int32_t*>(zsm + L.idx);
    uint16_t* s_inv = reinterpret_cast<uint16_t*>(zsm + L.inv);
    uint8_t* s_z = reinterpret_cast<uint8_t*>(zsm + L.z);
    uint16_t* cnt = reinterpret_cast<uint16_t*>(zsm + L.cnt);
    // each thread writes the source positions of its own pieces into s_idx;
    // the staging loop reads its element's slot before the cp.async that
    // overwrites it with the particle index
    if (per <= 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lo + u < hi) {
                const int c = e_[u] - a_[u], src0 = (lo + u) * tile + a_[u];
                for (int k = 0; k < c; ++k) s_idx[run + k] = src0 + k;
                run += c;
            }
    } else {
        for (int t = lo; t < hi; ++t) {
            const int a = __ldg(toff + (int64_t)t * (ncol + 1) + col);
            const int c = __ldg(toff + (int64_t)t * (ncol + 1) + col + 1) - a, src0 = t * tile + a;
            for (int k = 0; k < c; ++k) s_idx[run + k] = src0 + k;
            run += c;
        }
    }
    for (int e = tid; e < K2 * kZThreads; e += kZThreads) cnt[e] = 0;
    __syncthreads();
    for (int j = tid; j < m; j += kZThreads) {
        const int src = s_idx[j];
        cp_async16_s(s_rec + j, rec2 + src);
        cp_async16_s(reinterpret_cast<char*>(s_rec + j) + 16, reinterpret_cast<const char*>(rec2 + src) + 16);
        cp_async4_s(s_idx + j, idx2 + src);
    }
    cp_async_wait_all();
    __syncthreads();
    z_whole_body<(ZB <= 6 ? ZB : 6)>(g, col, cs, m, n, s_rec, s_idx, s_inv, s_z, cnt, perm, start, sp,
                                     wsum);
}

// ---- key path: the tile pass moves (particle, c2) pairs, not records ----------
// k_tile_keys   the tile pass of k_tile_sort reading only x, y, z (24 B per
//               particle) and writing 8-byte (particle, c2) pairs: the tile's
//               shared-memory stage is a fifth of the record path's
// k_z_tiles_ko  the column pass on pairs (one 8-byte cp.async per element);
//               the sorted records are gathered from the input arrays, which
//               the tile pass has just brought into L2, straight into sp
// The order, cell starts and records are identical to the record path.
struct TileKeysLayout {
    size_t pair, wc, tc, cb, total;
    __host__ __device__ TileKeysLayout(int ncol, int tile) {
        pair = 0;
        wc = pair + sizeof(int2) * tile;
        tc = wc + ((sizeof(uint16_t) * kTileWarps * ncol + 15) & ~size_t(15));
        cb = tc + sizeof(int32_t) * ncol;
        total = cb + sizeof(int32_t) * (ncol + 1);
    }
};

#ifndef KEYS_MINB
#define KEYS_MINB 4  // 64 registers, four tiles per SM (config 3: sort stage 59.8 -> 55.4 us with ZKO_MINB 3)
#endif
#ifndef ZKO_MINB
#define ZKO_MINB 3
#endif
template <int CB, int TR>
__global__ void __launch_bounds__(kTileWarps * 32, KEYS_MINB) k_tile_keys(Geometry g, int64_t n,
                                                               const double* __restrict__ xyz,
                                                               int32_t* __restrict__ toff,
                                                               int2* __restrict__ pairs,
                                                               unsigned long long* bad) {
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ int32_t wsum[32];
    const int ncol = g.K[0] * g.K[1];
    constexpr int kTT = TR * 32 * kTileWarps;
    const TileKeysLayout TL(ncol, kTT);
    int2* s_pair = reinterpret_cast<int2*>(tsm + TL.pair);
    uint16_t* wc = reinterpret_cast<uint16_t*>(tsm + TL.wc);  // [kTileWarps][ncol]
    int32_t* tc = reinterpret_cast<int32_t*>(tsm + TL.tc);
    int32_t* cb = reinterpret_cast<int32_t*>(tsm + TL.cb);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    TRACE_MARK(0, 0);
    pdl_trigger();  // the column pass may become resident
    for (int e = tid; e < (int)((TL.tc - TL.wc) / 16); e += blockDim.x)
        reinterpret_cast<uint4*>(wc)[e] = make_uint4(0u, 0u, 0u, 0u);
    const int64_t tbase = (int64_t)blockIdx.x * kTT;
    const int64_t wbase = tbase + w * (TR * 32);
    double px[TR], py[TR], pz[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {  // every load of the warp's slice in flight
        const int64_t i = wbase + r * 32 + lane;
        if (i < n) {
            // three 8-byte loads per particle; a 128-bit + 64-bit pair chosen on the
            // address (as in gather_rec) measured slower here: 50.6 vs 49.0 us sort stage
            px[r] = __ldg(xyz + 3 * i);
            py[r] = __ldg(xyz + 3 * i + 1);
            pz[r] = __ldg(xyz + 3 * i + 2);
        }
    }
    const double b = __dmul_rn(2.0, g.radius), y = g.inv_diam;
    int colr[TR], c2r[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        colr[r] = -1;
        c2r[r] = 0;
        if (i < n) {
            const double p0 = px[r], p1 = py[r], p2 = pz[r];
            if (fabs(p0 - g.center[0]) > g.radius || fabs(p1 - g.center[1]) > g.radius ||
                fabs(p2 - g.center[2]) > g.radius)
                atomicMin(&bad[0], (unsigned long long)i);  // Box3::contains (geometry.hpp:36-40)
            const int c0 = axis_cell2(p0, g.center[0], g.radius, g.K[0], b, y);
            const int c1 = axis_cell2(p1, g.center[1], g.radius, g.K[1], b, y);
            const int c2 = axis_cell2(p2, g.center[2], g.radius, g.K[2], b, y);
            if (c0 < g.x_lo || c0 >= g.x_hi || c1 < g.y_lo || c1 >= g.y_hi || c2 < g.z_lo || c2 >= g.z_hi)
                atomicOr(&bad[1], 2ull);  // not in this plan's cell block
            colr[r] = c0 * g.K[1] + c1;
            c2r[r] = c2;
        }
    }
    __syncthreads();
    TRACE_MARK(0, 1);
    unsigned pk[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const bool act = colr[r] >= 0;
        const int col = act ? colr[r] : -1 - lane;
        const unsigned peers = warp_peers<CB>(col);
        pk[r] = peers;
        if (act && lane == __ffs(peers) - 1) wc[w * ncol + col] += (uint16_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    TRACE_MARK(0, 2);
    for (int c = tid; c < ncol; c += blockDim.x) {
        int run = 0;
#pragma unroll
        for (int k = 0; k < kTileWarps; ++k) {
            const int t = wc[k * ncol + c];
            wc[k * ncol + c] = (uint16_t)run;
            run += t;
        }
        tc[c] = run;
    }
    __syncthreads();
    block_col_bases(tc, ncol, cb, wsum);
    TRACE_MARK(0, 3);
    // column-major offsets toff[c][tile]: a column CTA of the second pass reads
    // its two rows as contiguous runs (one scattered 4-byte store per column here)
    for (int c = tid; c <= ncol; c += blockDim.x) toff[(int64_t)c * gridDim.x + blockIdx.x] = cb[c];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const bool act = colr[r] >= 0;
        const unsigned peers = pk[r];
        int base = 0;
        if (act) base = cb[colr[r]] + wc[w * ncol + colr[r]];
        __syncwarp();
        if (act) {
            if (lane == __ffs(peers) - 1) wc[w * ncol + colr[r]] += (uint16_t)__popc(peers);
            const int pos = base + __popc(peers & ((1u << lane) - 1));
            s_pair[pos] = make_int2((int32_t)(wbase + r * 32 + lane), c2r[r]);
        }
        __syncwarp();
    }
    __syncthreads();
    TRACE_MARK(0, 4);
    const int tn = cb[ncol];
    for (int k = tid; k < tn; k += blockDim.x) pairs[tbase + k] = s_pair[k];
    TRACE_MARK(0, 5);
}

__device__ __forceinline__ void cp_async8_s(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Whole-column layout of the key path: pairs, inverse order, c2, counters.
struct ZPairsLayout {
    size_t pair, inv, z, cnt, total;
    __host__ __device__ ZPairsLayout(int K2, int cap) {
        pair = 0;
        inv = sizeof(int2) * cap;
        z = inv + sizeof(uint16_t) * cap;
        cnt = z + sizeof(uint8_t) * cap;
        cnt = (cnt + 15) & ~size_t(15);
        total = cnt + sizeof(uint16_t) * (size_t)K2 * kZThreads;
    }
};
// 4-bit per-thread counters: at most 15 of a thread's slice in one cell
constexpr int kZPairsCap = 15 * kZThreads;
__host__ inline int pairs_cap_for(int K2) {
    if (K2 > 64) return 0;
    for (int cap = kZPairsCap; cap >= 1024; cap -= 256)
        if (ZPairsLayout(K2, cap).total <= kZWholeMaxSmem) return cap;
    return 0;
}

template <int ZB>
__global__ void __launch_bounds__(kZThreads, ZKO_MINB) k_z_tiles_ko(Geometry g, int64_t n, int ntiles, int tile,
                                                           int whole_cap,
                                                           const int32_t* __restrict__ toff,
                                                           const int2* __restrict__ pairs,
                                                           const double* __restrict__ xyz,
                                                           const double* __restrict__ q,
                                                           int32_t* __restrict__ perm,
                                                           int32_t* __restrict__ start,
                                                           double4* __restrict__ sp) {
    extern __shared__ __align__(16) unsigned char zsm[];
    __shared__ int32_t wsum[32];
    const int col = blockIdx.x, ncol = g.K[0] * g.K[1], K2 = g.K[2];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int per = (ntiles + kZThreads - 1) / kZThreads;
    const int lo = min(ntiles, tid * per), hi = min(ntiles, lo + per);
    TRACE_MARK(1, 0);
    pdl_trigger();  // the spread may become resident
    pdl_wait();     // the tile pass's offsets and pairs
    int a_[4], e_[4];
    int csum = 0, psum = 0;
    if (per <= 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lo + u < hi) {
                a_[u] = __ldg(toff + (int64_t)col * ntiles + lo + u);
                e_[u] = __ldg(toff + (int64_t)(col + 1) * ntiles + lo + u);
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lo + u < hi) {
                csum += a_[u];
                psum += e_[u] - a_[u];
            }
    } else {
        for (int t = lo; t < hi; ++t) {
            const int a = __ldg(toff + (int64_t)col * ntiles + t);
            csum += a;
            psum += __ldg(toff + (int64_t)(col + 1) * ntiles + t) - a;
        }
    }
    int x = psum, cx = csum;
    for (int o = 1; o < 32; o <<= 1) {
        const int y1 = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y1;
        cx += __shfl_xor_sync(0xffffffffu, cx, o);
    }
    if (lane == 31) wsum[w] = x;
    if (lane == 0) wsum[16 + w] = cx;
    __syncthreads();
    int off = 0, cs = 0;
    for (int k = 0; k < kZWarps; ++k) {
        off += k < w ? wsum[k] : 0;
        cs += wsum[16 + k];
    }
    int m = 0;
    for (int k = 0; k < kZWarps; ++k) m += wsum[k];
    const bool whole = ZB <= 6 && m <= whole_cap;  // uniform per CTA
    int run = off + x - psum;
    if (!whole) {  // piece tables, binary-searched per element (chunked column sort)
        const ZTilesLayout TLc(K2, ntiles, 0);
        int32_t* pre = reinterpret_cast<int32_t*>(zsm + TLc.tables);
        int32_t* srca = pre + ntiles + 1;
        for (int t = lo; t < hi; ++t) {
            const int a = __ldg(toff + (int64_t)col * ntiles + t);
            srca[t] = t * tile + a;
            pre[t] = run;
            run += __ldg(toff + (int64_t)(col + 1) * ntiles + t) - a;
        }
        if (tid == 0) pre[ntiles] = m;
        __syncthreads();
        z_sort_chunked_acc<ZB>(g, col, cs, m, PieceSrc{pre, srca, ntiles}, PairAcc{pairs, xyz, q}, n, perm,
                               start, sp, zsm);
        return;
    }
    TRACE_MARK(1, 1);
    const ZPairsLayout L(K2, whole_cap);
    int2* s_pair = reinterpret_cast<int2*>(zsm + L.pair);
    uint16_t* s_inv = reinterpret_cast<uint16_t*>(zsm + L.inv);
    uint8_t* s_z = reinterpret_cast<uint8_t*>(zsm + L.z);
    uint16_t* cnt = reinterpret_cast<uint16_t*>(zsm + L.cnt);
    // every thread copies its own pieces, in tile order (ascending particles)
    if (per <= 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lo + u < hi) {
                const int c = e_[u] - a_[u];
                const int64_t src0 = (int64_t)(lo + u) * tile + a_[u];
                for (int k = 0; k < c; ++k) cp_async8_s(s_pair + run + k, pairs + src0 + k);
                run += c;
            }
    } else {
        for (int t = lo; t < hi; ++t) {
            const int a = __ldg(toff + (int64_t)col * ntiles + t);
            const int c = __ldg(toff + (int64_t)(col + 1) * ntiles + t) - a;
            const int64_t src0 = (int64_t)t * tile + a;
            for (int k = 0; k < c; ++k) cp_async8_s(s_pair + run + k, pairs + src0 + k);
            run += c;
        }
    }
    for (int e = tid; e < K2 * kZThreads; e += kZThreads) cnt[e] = 0;
    cp_async_wait_all();
    __syncthreads();
    TRACE_MARK(1, 2);
    z_whole_pairs<(ZB <= 6 ? ZB : 6)>(g, col, cs, m, n, s_pair, s_inv, s_z, cnt, perm, start, xyz, q, sp,
                                      wsum);
    TRACE_MARK(1, 6);
}

// Instantiation for an even key width in [2, 16].
template <class F>
auto pick_bits(int b, F f) {
    switch (b) {
        case 2: return f(std::integral_constant<int, 2>{});
        case 4: return f(std::integral_constant<int, 4>{});
        case 6: return f(std::integral_constant<int, 6>{});
        case 8: return f(std::integral_constant<int, 8>{});
        case 10: return f(std::integral_constant<int, 10>{});
        case 12: return f(std::integral_constant<int, 12>{});
        case 14: return f(std::integral_constant<int, 14>{});
        default: return f(std::integral_constant<int, 16>{});
    }
}

}  // namespace

bool sort2_supported(const Geometry& g) {
    const int ncol = g.K[0] * g.K[1];
    return ncol <= 32768 && (size_t)(kTileWarps * ncol + ncol + 1) * sizeof(int32_t) <= 160 * 1024 &&
           ZLayout(g.K[2]).total <= 160 * 1024 && g.K[2] <= 65536;
}

size_t sort2_hist_entries(const Geometry& g, int64_t cap) {  // also the tile path's toff
    const int64_t ntiles = (cap + kMinTile - 1) / kMinTile;
    return ((size_t)g.K[0] * g.K[1] + 1) * (size_t)std::max<int64_t>(1, ntiles);
}

// Variant choice. The tile path wins while a tile's piece of a column holds
// a few particles on average (config 2, ~17: 38.3 -> 28.4 us; config 3, ~5:
// 70.1 -> 64.1 us); with ~1 (config 4) the per-tile column tables dominate
// (308 vs 234 us). KPME_SORT_TILES=0 / 1 forces the column scatter / the tile
// path wherever it fits (tests, A/B).
static bool tiles_chosen(int ncol) {
    static const int m = [] {
        const char* e = getenv("KPME_SORT_TILES");
        return (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 1 : 2;
    }();
    return m == 1 || (m == 2 && ncol * 4 <= kTile);
}

template <class F>
auto pick_rounds(int tr, F f) {
    switch (tr) {
        case 4: return f(std::integral_constant<int, 4>{});
        case 7: return f(std::integral_constant<int, 7>{});
        default: return f(std::integral_constant<int, 8>{});
    }
}

static bool launch_sort2_tiles(const Geometry& g, int64_t n, const double* xyz, const SortBuffers& b,
                               cudaStream_t s, int* launches, const double* q, double4* sp) {
    const int ncol = g.K[0] * g.K[1];
    if (!tiles_chosen(ncol)) return false;
    // Tile rounds: the fewest (waves x tile length) at two CTAs per SM, among
    // tiles holding >= 4 particles per column on average (the pieces k_z_tiles
    // gathers); ties go to the longer tile. Config 3: 559 tiles of 1792.
    static const bool keys_on = [] {
        const char* e = getenv("KPME_SORT_KEYS");
        return !(e && *e == '0');
    }();
    const int slots = (keys_on && (q || !sp) ? KEYS_MINB : 2) * sm_count();
    int tr = 8;
    {
        int64_t best = -1;
        for (int cand : {8, 7, 4}) {
            const int tile = cand * 32 * kTileWarps;
            if (tile < 4 * ncol) continue;
            const int64_t nt = std::max<int64_t>(1, (n + tile - 1) / tile);
            const int64_t cost = (nt + slots - 1) / slots * cand;
            if (best < 0 || cost < best) {
                best = cost;
                tr = cand;
            }
        }
    }
    const int tile = tr * 32 * kTileWarps;
    const int ntiles = (int)std::max<int64_t>(1, (n + tile - 1) / tile);
    const TileLayout TL(ncol, tile);
    const int wcap = whole_cap_for(g.K[2]);
    const ZTilesLayout ZL(g.K[2], ntiles, wcap);
    if (TL.total > kTileMaxSmem || ntiles > 65535 || ZL.total_chunked > 160 * 1024) return false;
    const int cb = (bits_for(ncol) + 1) & ~1, zb = (bits_for(g.K[2]) + 1) & ~1;
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        for (int bb = 2; bb <= 16; bb += 2) {
            for (int r : {4, 7, 8})
                KB_CUDA(cudaFuncSetAttribute(pick_bits(bb, [r](auto B) {
                                                 return pick_rounds(r, [](auto T) {
                                                     return &k_tile_sort<decltype(B)::value, decltype(T)::value>;
                                                 });
                                             }),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileMaxSmem));
            KB_CUDA(cudaFuncSetAttribute(pick_bits(bb, [](auto B) { return &k_z_tiles<decltype(B)::value>; }),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        }
    });
    int l = 0;
    // Key path (default): the tile pass moves 8-byte (particle, c2) pairs and
    // the column pass gathers the records from the inputs. KPME_SORT_KEYS=0:
    // the record path.
    static const bool keys_env = [] {
        const char* e = getenv("KPME_SORT_KEYS");
        return !(e && *e == '0');
    }();
    const int pcap = pairs_cap_for(g.K[2]);
    const TileKeysLayout TK(ncol, tile);
    const ZTilesLayout ZLc(g.K[2], ntiles, 0);
    const size_t kzsmem = std::max(ZLc.total_chunked, pcap ? ZPairsLayout(g.K[2], pcap).total : 0);
    if (keys_env && (q || !sp) && TK.total <= kTileMaxSmem && kzsmem <= 160 * 1024) {
        static PerDevice keys_once;
        once_per_device(keys_once, [&] {
            for (int bb = 2; bb <= 16; bb += 2) {
                for (int r : {4, 7, 8})
                    KB_CUDA(cudaFuncSetAttribute(pick_bits(bb, [r](auto B) {
                                                     return pick_rounds(r, [](auto T) {
                                                         return &k_tile_keys<decltype(B)::value, decltype(T)::value>;
                                                     });
                                                 }),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileMaxSmem));
                KB_CUDA(cudaFuncSetAttribute(pick_bits(bb, [](auto B) { return &k_z_tiles_ko<decltype(B)::value>; }),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
            }
        });
        int2* pairs = reinterpret_cast<int2*>(b.rec);
        if (n > 0) {
            auto tk = pick_bits(cb, [tr](auto B) {
                return pick_rounds(tr, [](auto T) { return &k_tile_keys<decltype(B)::value, decltype(T)::value>; });
            });
            tk<<<ntiles, kTileWarps * 32, TK.total, s>>>(g, n, xyz, b.hist, pairs, b.bad);
            KB_CHECK_LAUNCH();
            ++l;
        } else {
            KB_CUDA(cudaMemsetAsync(b.hist, 0, sizeof(int32_t) * (ncol + 1), s));
        }
        auto zk = pick_bits(zb, [](auto B) { return &k_z_tiles_ko<decltype(B)::value>; });
#ifdef ZKO_NOSP  // profiling ablation only: no record write-out (results invalid)
        sp = nullptr;
#endif
        launch_pdl_if((pdl_mask() & 1) != 0, zk, dim3(ncol), dim3(kZThreads), kzsmem, s, g, n, ntiles, tile, pcap, b.hist, pairs, xyz, q,
                   b.perm, b.start, sp);
        KB_CHECK_LAUNCH();
        if (launches) *launches += l + 1;
        return true;
    }
    auto tile_kernel = pick_bits(cb, [tr](auto B) {
        return pick_rounds(tr, [](auto T) { return &k_tile_sort<decltype(B)::value, decltype(T)::value>; });
    });
    auto z_kernel = pick_bits(zb, [](auto B) { return &k_z_tiles<decltype(B)::value>; });
    if (n > 0) {
        tile_kernel<<<ntiles, kTileWarps * 32, TL.total, s>>>(g, n, xyz, q, b.hist, b.idx2, b.rec, b.bad);
        KB_CHECK_LAUNCH();
        ++l;
    } else {
        KB_CUDA(cudaMemsetAsync(b.hist, 0, sizeof(int32_t) * (ncol + 1), s));
    }
    const int whole_cap = wcap > 0 && ZL.total_whole <= kZWholeMaxSmem ? wcap : 0;
    const size_t zsmem = std::max(ZL.total_chunked, whole_cap ? ZL.total_whole : 0);
    z_kernel<<<ncol, kZThreads, zsmem, s>>>(g, n, ntiles, tile, whole_cap, b.hist, b.idx2, b.rec, b.perm,
                                            b.start, sp);
    KB_CHECK_LAUNCH();
    ++l;
    if (launches) *launches += l;
    return true;
}

void launch_sort2(const Geometry& g, int64_t n, const double* xyz, const SortBuffers& b,
                  cudaStream_t s, int* launches, const double* q, double4* sp) {
    if (!q) sp = nullptr;
    if (launch_sort2_tiles(g, n, xyz, b, s, launches, q, sp)) return;
    // key widths rounded up to an even bit count (extra ballots see zero bits)
    const int ncol = g.K[0] * g.K[1];
    const int cb = (bits_for(ncol) + 1) & ~1, zb = (bits_for(g.K[2]) + 1) & ~1;
    auto col_kernel = pick_bits(cb, [](auto B) { return &k_col_scatter<decltype(B)::value>; });
    auto z_kernel = pick_bits(zb, [](auto B) { return &k_z_sort<decltype(B)::value>; });
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        for (int b = 2; b <= 16; b += 2) {
            KB_CUDA(cudaFuncSetAttribute(pick_bits(b, [](auto B) { return &k_col_scatter<decltype(B)::value>; }),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
            KB_CUDA(cudaFuncSetAttribute(pick_bits(b, [](auto B) { return &k_z_sort<decltype(B)::value>; }),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        }
        KB_CUDA(cudaFuncSetAttribute(k_tile_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     160 * 1024));
    });
    const int ntiles = (int)std::max<int64_t>(1, (n + kTile - 1) / kTile);
    const int64_t E = (int64_t)ncol * ntiles;
    int l = 0;
    if (n > 0) {
        k_tile_hist<<<ntiles, kHistThreads, ncol * sizeof(int32_t), s>>>(g, n, xyz, b.key, b.hist,
                                                                          ntiles, b.bad);
        ++l;
    } else {
        KB_CUDA(cudaMemsetAsync(b.hist, 0, sizeof(int32_t) * E, s));
    }
    KB_CHECK_LAUNCH();
    k_col_scan<<<(ncol + 7) / 8, 256, 0, s>>>(ncol, ntiles, b.hist, b.ctot, b.cbase, b.ticket);
    KB_CHECK_LAUNCH();
    ++l;
    if (n > 0) {
        col_kernel<<<ntiles, kTileWarps * 32, ((kTileWarps * ncol + 1) / 2 + ncol) * sizeof(int32_t),
                        s>>>(g, n, ntiles, b.key, b.hist, b.cbase, xyz, q, b.idx2, b.rec);
        KB_CHECK_LAUNCH();
        ++l;
    }
    const int whole_cap = whole_cap_for(g.K[2]);
    const size_t zsmem = std::max(ZLayout(g.K[2]).total,
                                  whole_cap ? ZWholeLayout(g.K[2], whole_cap).total : 0);
    z_kernel<<<ncol, kZThreads, zsmem, s>>>(g, b.cbase, n, whole_cap, b.idx2, b.rec, b.perm,
                                            b.start, sp);
    KB_CHECK_LAUNCH();
    ++l;
    if (launches) *launches += l;
}

}  // namespace kb

TRACE_READER(sort2)
