// dense.cu -- the dense SKP grid operator y = sum_r (A_r (x) B_r (x) C_r) x on
// FP64 DMMA tensor cores (config 5; kron_matvec_shuffle semantics,
// kron.hpp:180-197, summed over terms as spkmv_sum does, parallel.hpp:193-196).
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects .kind::f64), so FP64 tensor
// work is warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4). Every mode product is
// one GEMM of the form
//     out[m][i] = sum_k in[k][m] * F[i][k]          (M x N, contraction K)
// which contracts the SLOWEST axis of a lexicographic tensor and appends the
// result as the FASTEST axis. Three such passes rotate the axes back to the
// original order: [x][y][z] -A-> [y][z][x'] -B-> [z][x'][y'] -C-> [x'][y'][z'].
// The last pass contracts over (term, z) at once (K = chunk * n2), so the
// per-term partial sums accumulate in the DMMA registers.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "internal.h"

namespace kb {
namespace {

constexpr int BM = 128, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int LDA = BM + 8;  // As[k][m]: row offsets alternate 0/64 B mod 128 -> no conflicts
constexpr int LDB = BK + 4;  // Bs[i][k]: row offsets step 32 B mod 128 -> no conflicts
constexpr size_t kSmem = sizeof(double) * STAGES * (BK * LDA + BN * LDB);

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid ? 8 : 0;  // zero-fill out-of-range elements
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int valid_doubles) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid_doubles * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// VEC16: all rows 16-byte aligned (M and K even, pointers aligned) -> 16-byte copies.
// blockIdx.z selects a batch entry: in += z * sin, F += z * sF, out += z * sout.
template <bool VEC16>
__global__ void __launch_bounds__(THREADS) k_dgemm_tn(int64_t M, int64_t N, int64_t K,
                                                      const double* __restrict__ in,
                                                      const double* __restrict__ F,
                                                      double* __restrict__ out, int accumulate,
                                                      int64_t sin, int64_t sF, int64_t sout) {
    in += blockIdx.z * sin;
    F += blockIdx.z * sF;
    out += blockIdx.z * sout;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                         // [STAGES][BK][LDA]
    double* Bs = smem + STAGES * BK * LDA;     // [STAGES][BN][LDB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;   // 2 x 2 warps, warp tile 64 x 32
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const int ktiles = (int)((K + BK - 1) / BK);

    auto load = [&](int stage, int kt) {
        double* as = As + stage * BK * LDA;
        double* bs = Bs + stage * BN * LDB;
        const int64_t k0 = (int64_t)kt * BK;
        if (VEC16) {
            for (int idx = tid; idx < BK * BM / 2; idx += THREADS) {
                const int kk = idx / (BM / 2), mm = (idx % (BM / 2)) * 2;
                const int64_t gk = k0 + kk, gm = m0 + mm;
                int v = (gk < K) ? (int)std::min<int64_t>(2, std::max<int64_t>(0, M - gm)) : 0;
                const double* src = in + (v ? gk * M + gm : 0);
                cp_async16(as + kk * LDA + mm, src, v);
            }
            for (int idx = tid; idx < BN * BK / 2; idx += THREADS) {
                const int ii = idx / (BK / 2), kk = (idx % (BK / 2)) * 2;
                const int64_t gi = n0 + ii, gk = k0 + kk;
                int v = (gi < N) ? (int)std::min<int64_t>(2, std::max<int64_t>(0, K - gk)) : 0;
                const double* src = F + (v ? gi * K + gk : 0);
                cp_async16(bs + ii * LDB + kk, src, v);
            }
        } else {
            for (int idx = tid; idx < BK * BM; idx += THREADS) {
                const int kk = idx / BM, mm = idx % BM;
                const int64_t gk = k0 + kk, gm = m0 + mm;
                const bool v = gk < K && gm < M;
                cp_async8(as + kk * LDA + mm, in + (v ? gk * M + gm : 0), v);
            }
            for (int idx = tid; idx < BN * BK; idx += THREADS) {
                const int ii = idx / BK, kk = idx % BK;
                const int64_t gi = n0 + ii, gk = k0 + kk;
                const bool v = gi < N && gk < K;
                cp_async8(bs + ii * LDB + kk, F + (v ? gi * K + gk : 0), v);
            }
        }
    };

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load(s, s);
        cp_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int nk = kt + STAGES - 1;
        if (nk < ktiles) load(nk % STAGES, nk);
        cp_commit();
        const double* as = As + (kt % STAGES) * BK * LDA + wm * 64 + (lane >> 2);
        const double* bs = Bs + (kt % STAGES) * BN * LDB + (wn * 32 + (lane >> 2)) * LDB;
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = as[(k4 + (lane & 3)) * LDA + i * 8];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = bs[j * 8 * LDB + k4 + (lane & 3)];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
        }
    }
    cp_wait<0>();

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = m0 + wm * 64 + i * 8 + (lane >> 2);
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t col = n0 + wn * 32 + j * 8 + 2 * (lane & 3);
#pragma unroll
            for (int c = 0; c < 2; ++c)
                if (col + c < N) {
                    double* o = out + row * N + col + c;
                    *o = accumulate ? *o + acc[i][j][c] : acc[i][j][c];
                }
        }
    }
}

// ---- TMA-staged variant ------------------------------------------------------
// The same 128 x 64 x 16 CTA tile and warp tiling, with operand tiles staged by
// the Tensor Memory Accelerator: one cp.async.bulk.tensor per operand per
// k-tile, issued by one thread, completing on an mbarrier per stage; out-of-
// range rows/columns arrive as zeros (no predicated per-element copies).
//   A tile: in[z][k][m], box {128 m, 16 k}, dense [16][128] (row offsets are
//           multiples of 1 KB, so the fragment reads of 4 k rows are 2-way
//           conflicted; they are 1/3 of the smem traffic per DMMA)
//   B tile: F[z][i][k], box {16 k, 64 i}, 128-byte swizzle: the 16-byte chunk
//           c of row i sits at chunk c ^ (i % 8), so a warp's fragment reads
//           (8 rows x 2 chunks per k pair) are conflict-free.
constexpr int TSTAGES = 4;
constexpr size_t kTmaA = (size_t)BK * BM * sizeof(double);  // 16 KB
constexpr size_t kTmaB = (size_t)BN * BK * sizeof(double);  // 8 KB
constexpr size_t kSmemTma = TSTAGES * (kTmaA + kTmaB) + 1024 + 64;

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbarrier_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbarrier_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbarrier_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tTMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TMA_WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

__global__ void __launch_bounds__(THREADS) k_dgemm_tn_tma(int64_t M, int64_t N, int64_t K,
                                                          const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB,
                                                          int zA, int zB, double* __restrict__ out,
                                                          int accumulate, int64_t sout) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // 1024-byte alignment for the 128-byte swizzle
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* As = reinterpret_cast<double*>(base);                       // [S][BK][BM]
    double* Bs = reinterpret_cast<double*>(base + TSTAGES * kTmaA);     // [S][BN][BK] swizzled
    uint64_t* full = reinterpret_cast<uint64_t*>(base + TSTAGES * (kTmaA + kTmaB));
    // grid (batch, m tile, n tile): the batch entries sharing an operand tile
    // (the broadcast mesh of the per-term passes) are scheduled together, so
    // the tile is read from DRAM once and served from L2 to the rest
    const int bz = blockIdx.x;
    out += bz * sout;
    const int za = zA ? bz : 0, zb = zB ? bz : 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.z * BN;
    const int ktiles = (int)((K + BK - 1) / BK);
    if (tid == 0) {
        for (int s = 0; s < TSTAGES; ++s) mbarrier_init(full + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int kt) {
        const int s = kt % TSTAGES;
        mbarrier_expect_tx(full + s, (unsigned)(kTmaA + kTmaB));
        tma_load_3d(As + (size_t)s * BK * BM, &tmA, (int)m0, kt * BK, za, full + s);
        tma_load_3d(Bs + (size_t)s * BN * BK, &tmB, kt * BK, (int)n0, zb, full + s);
    };
    if (tid == 0)
        for (int kt = 0; kt < TSTAGES && kt < ktiles; ++kt) issue(kt);

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int g = lane >> 2, c = lane & 3;
    for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % TSTAGES;
        mbarrier_wait(full + s, (unsigned)((kt / TSTAGES) & 1));
        const double* as = As + (size_t)s * BK * BM + wm * 64 + g;
        const char* bs = reinterpret_cast<const char*>(Bs + (size_t)s * BN * BK);
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = as[(k4 + c) * BM + i * 8];
            const int kk = k4 + c;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int row = wn * 32 + j * 8 + g;  // row % 8 == g
                b[j] = *reinterpret_cast<const double*>(
                    bs + row * 128 + ((((kk >> 1) ^ g) & 7) << 4) + ((kk & 1) << 3));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
        }
        __syncthreads();  // stage s fully read
        if (tid == 0 && kt + TSTAGES < ktiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(kt + TSTAGES);
        }
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = m0 + wm * 64 + i * 8 + g;
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t col = n0 + wn * 32 + j * 8 + 2 * c;
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (col + e < N) {
                    double* o = out + row * N + col + e;
                    *o = accumulate ? *o + acc[i][j][e] : acc[i][j][e];
                }
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// rows x cols (cols fastest) x batch FP64 tensor; batch stride in elements
// (0: one matrix broadcast to every batch entry).
bool make_map(CUtensorMap* map, const double* ptr, int64_t rows, int64_t cols, int64_t bstride,
              int batch, unsigned box_cols, unsigned box_rows, bool swizzle128) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows,
                                (cuuint64_t)(bstride ? batch : 1)};
    const cuuint64_t strides[2] = {(cuuint64_t)cols * 8, (cuuint64_t)(bstride ? bstride : rows * cols) * 8};
    const cuuint32_t box[3] = {box_cols, box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// out[e] (+)= sum_s part[s][e] over splits in order (deterministic split-K).
__global__ void k_sum_splits(int64_t E, int splits, const double* __restrict__ part,
                             double* __restrict__ out, int accumulate) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        double s = accumulate ? out[e] : 0.0;
        for (int k = 0; k < splits; ++k) s += part[(int64_t)k * E + e];
        out[e] = s;
    }
}

// Ccat[z'][r * nzi + z] = C_r[z'][coff + z] (z' < n2o, C_r row stride ldc):
// the term-concatenated last-pass operand (a column slice of C for slabs).
__global__ void k_concat_terms(int nterms, int n2o, int nzi, int ldc, int coff,
                               const double* __restrict__ C, double* __restrict__ Ccat) {
    const int64_t total = (int64_t)nterms * n2o * nzi;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(e % nzi), zp = (int)((e / nzi) % n2o), r = (int)(e / ((int64_t)nzi * n2o));
        Ccat[(int64_t)zp * nterms * nzi + (int64_t)r * nzi + z] =
            C[((int64_t)r * n2o + zp) * ldc + coff + z];
    }
}

// Ccat[k][z'][r' nzi + z] = C_{k tps + r'}[z'][coff + z]: the term-concatenated
// last-pass operand of every split k (tps terms each) in one launch.
__global__ void k_concat_splits(int nterms, int tps, int n2o, int nzi, int ldc, int coff,
                                const double* __restrict__ C, double* __restrict__ Ccat) {
    const int64_t total = (int64_t)nterms * n2o * nzi;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(e % nzi), zp = (int)((e / nzi) % n2o), r = (int)(e / ((int64_t)nzi * n2o));
        const int k = r / tps, rl = r % tps;
        Ccat[(int64_t)k * tps * n2o * nzi + (int64_t)zp * tps * nzi + (int64_t)rl * nzi + z] =
            C[((int64_t)r * n2o + zp) * ldc + coff + z];
    }
}

// Largest divisor of cr not above want: equal term counts per split, so the
// split GEMMs are one batched launch.
int even_splits(int want, int cr) {
    for (int d = std::min(want, cr); d > 1; --d)
        if (cr % d == 0) return d;
    return 1;
}

int chunk_terms(int n0, int n1, int n2, int nterms) {
    // keep the term-stacked intermediates (two per term) within ~16 GB of HBM
    const double mesh = 8.0 * n0 * n1 * n2;
    int c = (int)std::max(1.0, std::min((double)nterms, 8e9 / mesh));
    return std::max(1, std::min(c, nterms));
}

// CTA tiles of one mode-product GEMM; below ~2 waves the passes are batched
// over terms and the last pass is split over terms.
int64_t tiles(int64_t M, int64_t N) { return ((M + BM - 1) / BM) * ((N + BN - 1) / BN); }
int splits_for(int n0, int n1, int n2, int chunk) {
    const int64_t t = tiles((int64_t)n0 * n1, n2);
    int s = (int)std::max<int64_t>(1, (2 * sm_count() + t - 1) / t);
    return std::max(1, std::min(s, chunk));
}

}  // namespace

void dgemm_tn_batched(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* in,
                      int64_t sin, const double* F, int64_t sF, double* out, int64_t sout,
                      int batch, bool accumulate);

void dgemm_tn(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* in, const double* F,
              double* out, bool accumulate) {
    dgemm_tn_batched(s, M, N, K, in, 0, F, 0, out, 0, 1, accumulate);
}

void dgemm_tn_batched(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* in,
                      int64_t sin, const double* F, int64_t sF, double* out, int64_t sout,
                      int batch, bool accumulate) {
    static PerDevice attr_once;
    once_per_device(attr_once, [&] {
        KB_CUDA(cudaFuncSetAttribute(k_dgemm_tn<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kSmem));
        KB_CUDA(cudaFuncSetAttribute(k_dgemm_tn<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    });
    if (M <= 0 || N <= 0 || batch <= 0) return;
    const dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)batch);
    // TMA path: 16-byte aligned bases and row / batch strides (M, K even)
    static const bool tma_env = [] {
        const char* e = getenv("KPME_DGEMM_TMA");
        return !(e && *e == '0');
    }();
    const bool tma_ok = tma_env && (M % 2 == 0) && (K % 2 == 0) && ((uintptr_t)in % 16 == 0) &&
                        ((uintptr_t)F % 16 == 0) && (sin % 2 == 0) && (sF % 2 == 0) &&
                        K < (int64_t(1) << 31) && grid.x <= 65535 && grid.y <= 65535;
    if (tma_ok) {
        CUtensorMap ta, tb;
        if (make_map(&ta, in, K, M, sin, batch, BM, BK, false) &&
            make_map(&tb, F, N, K, sF, batch, BK, BN, true)) {
            static PerDevice tma_once;
            once_per_device(tma_once, [&] {
                KB_CUDA(cudaFuncSetAttribute(k_dgemm_tn_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemTma));
            });
            const dim3 tgrid((unsigned)batch, grid.x, grid.y);
            k_dgemm_tn_tma<<<tgrid, THREADS, kSmemTma, s>>>(M, N, K, ta, tb, sin ? 1 : 0, sF ? 1 : 0,
                                                           out, accumulate ? 1 : 0, sout);
            KB_CHECK_LAUNCH();
            return;
        }
    }
    const bool vec = (M % 2 == 0) && (K % 2 == 0) && ((uintptr_t)in % 16 == 0) &&
                     ((uintptr_t)F % 16 == 0) && (sin % 2 == 0) && (sF % 2 == 0);
    if (vec)
        k_dgemm_tn<true><<<grid, THREADS, kSmem, s>>>(M, N, K, in, F, out, accumulate ? 1 : 0, sin,
                                                      sF, sout);
    else
        k_dgemm_tn<false><<<grid, THREADS, kSmem, s>>>(M, N, K, in, F, out, accumulate ? 1 : 0,
                                                       sin, sF, sout);
    KB_CHECK_LAUNCH();
}

size_t kron_local_workspace_bytes(int n0, int n1, int nzi, int n2o, int nterms) {
    const size_t mi = (size_t)n0 * n1 * nzi, mo = (size_t)n0 * n1 * n2o;
    const int c = chunk_terms(n0, n1, std::max(nzi, n2o), nterms);
    const int sp = splits_for(n0, n1, n2o, c);
    return sizeof(double) * (mi * 2 * (size_t)c + (sp > 1 ? mo * sp : 0) + (size_t)n2o * nzi * c) + 256;
}

size_t dense_workspace_bytes(int n0, int n1, int n2, int nterms) {
    return kron_local_workspace_bytes(n0, n1, n2, n2, nterms);
}

void kron_local(cudaStream_t s, int n0, int n1, int nzi, int n2o, int nterms, const double* A,
                const double* B, const double* C, int ldc, int coff, const double* x, double* y,
                bool accumulate, double* work, size_t work_bytes) {
    const int64_t mi = (int64_t)n0 * n1 * nzi, mo = (int64_t)n0 * n1 * n2o;
    if (nterms <= 0 || nzi <= 0) {
        if (!accumulate) KB_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * mo, s));
        return;
    }
    const int chunk = chunk_terms(n0, n1, std::max(nzi, n2o), nterms);
    const int splits = splits_for(n0, n1, n2o, chunk);
    if (work_bytes < kron_local_workspace_bytes(n0, n1, nzi, n2o, nterms))
        throw Error(KPME_GPU_INVALID_ARGUMENT, "kron_matvec_dense: workspace too small");
    double* t1 = work;                          // [chunk][n1][nzi][n0]
    double* t2 = t1 + mi * chunk;               // [chunk][nzi][n0][n1]
    double* ccat = t2 + mi * chunk;             // [n2o][chunk * nzi]
    double* part = ccat + (int64_t)n2o * nzi * chunk;  // [splits][n0 n1][n2o]
    for (int r0 = 0; r0 < nterms; r0 += chunk) {
        const int cr = std::min(chunk, nterms - r0);
        const bool acc = accumulate || r0 > 0;
        // pass A, all terms of the chunk in one launch: t1_r = x ^T-contracted with A_r
        dgemm_tn_batched(s, (int64_t)n1 * nzi, n0, n0, x, 0, A + (int64_t)r0 * n0 * n0,
                         (int64_t)n0 * n0, t1, mi, cr, false);
        // pass B: t2_r[(z,x')][y'] = sum_y t1_r[y][(z,x')] B_r[y'][y]
        dgemm_tn_batched(s, (int64_t)nzi * n0, n1, n1, t1, mi, B + (int64_t)r0 * n1 * n1,
                         (int64_t)n1 * n1, t2, mi, cr, false);
        // pass C over (term, z): y[(x',y')][z'] (+)= sum_{r,z} t2[r][z][(x',y')] C_r[z'][coff + z]
        const double* Cr = C + (int64_t)r0 * n2o * ldc;
        const int sp = even_splits(splits, cr);
        if (sp <= 1) {
            k_concat_terms<<<sm_count() * 4, 256, 0, s>>>(cr, n2o, nzi, ldc, coff, Cr, ccat);
            KB_CHECK_LAUNCH();
            dgemm_tn(s, (int64_t)n0 * n1, n2o, (int64_t)cr * nzi, t2, ccat, y, acc);
        } else {
            // split-K over terms, one batched launch: split k covers terms
            // [k tps, (k+1) tps) with its concatenated operand [z'][tps nzi]
            // at ccat + k tps n2o nzi; partial sums summed in split order below
            const int tps = cr / sp;
            k_concat_splits<<<sm_count() * 4, 256, 0, s>>>(cr, tps, n2o, nzi, ldc, coff, Cr, ccat);
            KB_CHECK_LAUNCH();
            dgemm_tn_batched(s, (int64_t)n0 * n1, n2o, (int64_t)tps * nzi, t2, tps * mi, ccat,
                             (int64_t)tps * n2o * nzi, part, mo, sp, false);
            k_sum_splits<<<sm_count() * 8, 256, 0, s>>>(mo, sp, part, y, acc ? 1 : 0);
            KB_CHECK_LAUNCH();
        }
    }
}

void kron_matvec_dense(cudaStream_t s, int n0, int n1, int n2, int nterms, const double* A,
                       const double* B, const double* C, const double* x, double* y, double* work,
                       size_t work_bytes) {
    kron_local(s, n0, n1, n2, n2, nterms, A, B, C, n2, 0, x, y, false, work, work_bytes);
}

}  // namespace kb
