// internal.h -- shared declarations of the sm_100a implementation behind
// include/kpme_gpu.h. Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

#include "kpme_gpu.h"

namespace kb {

// Status-carrying exception used inside the library; the C-ABI layer maps it
// to a return code + kpme_gpu_last_error().
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define KB_CUDA(call)                                                               \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess)                                                      \
            throw ::kb::Error(KPME_GPU_CUDA, std::string(#call) + ": " +            \
                                                 cudaGetErrorString(e_));           \
    } while (0)

#define KB_CHECK_LAUNCH() KB_CUDA(cudaGetLastError())

// One-time setup per device (cudaFuncSetAttribute of kernels using more than
// 48 KB of dynamic shared memory). Function attributes are per device, plans
// may live on several devices of one process and be created from several
// host threads, so a process-wide flag is not enough.
struct PerDevice {
    static constexpr int kMax = 64;
    std::once_flag flag[kMax];
};
inline int current_device() {
    int d = 0;
    KB_CUDA(cudaGetDevice(&d));
    if (d < 0 || d >= PerDevice::kMax) throw Error(KPME_GPU_CUDA, "device ordinal out of range");
    return d;
}
template <class F>
inline void once_per_device(PerDevice& pd, F&& f) {
    std::call_once(pd.flag[current_device()], std::forward<F>(f));
}
// SM count of the current device (cached per device, thread-safe).
int sm_count();

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// start while its predecessor in the stream is still running, once every CTA
// of the predecessor has executed pdl_trigger() (or exited); it must call
// pdl_wait() before touching anything ANY earlier kernel of the chain writes:
// every kernel triggers when it starts, so a kernel can be resident while a
// kernel several links back is still running, and only plan constants (the
// W tables, G, the cell axes) may be read before the wait. The column
// kernels use it so that a kernel's CTAs are resident, and its table loads
// done, when the grid-wide dependency (the summed core) arrives. Both device
// calls are no-ops in a kernel launched the ordinary way. KPME_PDL=0 launches
// everything the ordinary way.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("KPME_PDL");
        return !(e && *e == '0');
    }();
    return on;
}
inline int pdl_mask() {  // debugging: KPME_PDL_MASK bit per launch site (1 z pass, 2 spread, 4 core sum, 8 gather)
    static const int m = [] {
        const char* e = getenv("KPME_PDL_MASK");
        return e ? atoi(e) : 15;
    }();
    return m;
}
// `on` = false launches the ordinary way (KPME_PDL_MASK, debugging).
template <class... KArgs, class... Args>
void launch_pdl_if(bool on, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = on && pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KB_CUDA(cudaLaunchKernelEx(&cfg, kern, KArgs(args)...));
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    launch_pdl_if(true, kern, grid, block, smem, s, args...);
}

// Makes `device` current for one ABI call and restores the caller's current
// device afterwards (the reference API has no device state to disturb).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device) {
        KB_CUDA(cudaGetDevice(&prev));
        if (prev != device) KB_CUDA(cudaSetDevice(device));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

#ifdef __CUDACC__
// 256-bit global accesses (one LDG/STG.E.ENL2.256 per particle record on
// sm_100a instead of two 128-bit ones: half the L2 requests for scattered
// record moves). Pointers are 32-byte aligned (double4 arrays).
__device__ __forceinline__ void st_rec(double4* p, const double4& v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z),
                 "d"(v.w)
                 : "memory");
}
// Cell index along one axis, bit-identical to the reference
// (geometry.hpp:141-148): t = ((p - (c - r)) * K) / (2 r), floor, face
// tie-break, clamp. The division is Markstein's correctly rounded quotient
// q = RN(q0 + (a - b q0) y) with b = 2r, y = RN(1/b), q0 = RN(a y) (exact FMA
// remainder), equal to RN(a / b) for these normal operands; the other
// operations are explicit round-to-nearest (no FMA contraction). Shared by
// every kernel that keys particles (sort, sort2, interp, route).
__device__ __forceinline__ int exact_axis_cell(double p, double c, double r, int K, double b,
                                               double y) {
    const double a = __dmul_rn(__dsub_rn(p, __dsub_rn(c, r)), (double)K);
    const double q0 = __dmul_rn(a, y);
    const double t = __fma_rn(__fma_rn(-q0, b, a), y, q0);
    int idx = (int)floor(t);
    if (t == (double)idx && idx > 0) --idx;
    return idx < 0 ? 0 : (idx > K - 1 ? K - 1 : idx);
}
__device__ __forceinline__ double4 ld_rec(const double4* p) {  // read-only data
    double4 v;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p));
    return v;
}
#endif

// Cell-grid geometry in the reference's terms (CellGrid, geometry.hpp:63-111)
// plus the derived sizes the kernels need. Passed to kernels by value.
struct Geometry {
    double center[3];
    double radius;
    int K[3];      // cells per axis
    int L;         // interpolation order (nodes per cell axis)
    int n[3];      // mesh points per axis, K_a * L (cell-face nodes duplicated)
    int M;         // modes
    int R;         // compacted Fourier rows per axis, 2M+1 (the m=0 sine row is 0)
    int ncell;     // K0*K1*K2
    int z_lo, z_hi;  // cell planes along axis 2 owned by this plan (slab)
    int x_lo, x_hi, y_lo, y_hi;  // cell ranges along axes 0, 1 (a block of a rank grid)
    double inv_diam; // RN(1 / (2 radius)), for the correctly rounded key division
};

// Columns (c0, c1) of the plan's cell block; column kernels launch
// block_columns * S CTAs.
inline int block_columns(const Geometry& g) { return (g.x_hi - g.x_lo) * (g.y_hi - g.y_lo); }

// ---- sort.cu ----------------------------------------------------------------
struct SortBuffers {
    int32_t* cnt;         // [ncell] histogram, then cursor
    int32_t* start;       // [ncell+1]
    int32_t* key;         // [n]
    int32_t* rank;        // [n] provisional slot within the cell
    int32_t* perm;        // [n]
    double4* rec;         // [n] particle records at their provisional slots
    // two-level counting sort (sort2.cu)
    int32_t* hist;        // [ncol * ntiles] per-tile column histogram, then its scan
    int32_t* ctot;        // [ncol] column totals
    int32_t* cbase;       // [ncol + 1] column starts
    unsigned* ticket;     // [1] last-CTA counter of k_col_scan (zero between launches)
    int32_t* idx2;        // [n + 4] column-ordered particle indices
    int32_t* big;         // [ncell] cells too large for the warp sorter
    int32_t* nbig;        // [1]
    unsigned long long* bad;  // [2]: lowest out-of-box index, out-of-cell flag
};
// Also writes the sorted particles sp (x, y, z, q) when q and sp are given.
void launch_sort(const Geometry& g, int64_t n, const double* xyz, const SortBuffers& b,
                 cudaStream_t s, int* launches, const double* q = nullptr, double4* sp = nullptr);
bool sort2_supported(const Geometry& g);
size_t sort2_hist_entries(const Geometry& g, int64_t cap);
void launch_sort2(const Geometry& g, int64_t n, const double* xyz, const SortBuffers& b,
                  cudaStream_t s, int* launches, const double* q = nullptr, double4* sp = nullptr);
void launch_permute(int64_t n, const double* xyz, const double* q, const int32_t* perm,
                    double4* sp, cudaStream_t s);

// ---- interp.cu --------------------------------------------------------------
// spread (+ forward z-contraction) per column of cells
struct ColumnArgs {
    Geometry g;
    const int32_t* start;
    const double4* sp;       // sorted particles (x, y, z, q)
    const double* W2;        // [R][n2]
    int S;                   // z segments per column
    double* T1;              // [S][n0][n1][R]
    double* colq;            // [S][K0*K1]
    double* phi_cells;       // optional out / in
    const double* B2;        // [n0][n1][R]
    double* psi_cells;       // optional out / in
    const double* corr;      // device scalar: c_Lambda * sum q (nullable)
    const int32_t* perm;     // sorted slot -> particle index
    double* out;             // potentials in particle order
    unsigned long long* bad;
    // fused core (hot path): spread writes per-column partial cores, gather
    // rebuilds its B2 block from the summed core
    const double* W0;        // [R][n0]
    const double* W1;        // [R][n1]
    double* Fpart;           // [R^3+1][fstride] partial cores (last entry: sum q)
    int fstride;             // Fpart row stride; 0 = S*K0*K1 (one particle chunk)
    const double* Gc;        // [R^3] collapsed SKP core
    const double* Fc;        // [R^3+1] summed core
    double correction;       // c_Lambda
    // monomial hot path: the W tables above are W_a Lambda (Lagrange basis ->
    // powers of the cell-local coordinate) and particles carry t^a, not w_k(t)
    int mono;
    // per-axis cell tables (axis_lo, axis_hi, midpoint, 1/half-width), K_a each
    const double4* cellax[3];
    // monomial gather: a thread takes two adjacent particles (pays off when
    // cells are full enough that a warp's pairs rarely straddle a cell)
    int gpairs;
    // direct records (hot path): the sort writes no sorted copy of the
    // particles; the spread and gather read record s as
    // (xyz[perm[s]], qv[perm[s]]) from the inputs, L2-resident after the sort
    int direct;
    const double* xyz;
    const double* qv;
};
enum SpreadMode { SPREAD_PARTICLES = 0, SPREAD_FROM_CELLS = 1 };
enum GatherMode { GATHER_FROM_B2 = 0, GATHER_FROM_CELLS = 1, PSI_ONLY = 2 };
void launch_spread_fwd(const ColumnArgs& a, int mode, bool want_fwd, cudaStream_t s);
// The kernels that read records through ColumnArgs::direct (the split-exponent
// spread and the monomial gather) serve this geometry.
bool direct_records_ok(const Geometry& g);
void launch_bwd_gather(const ColumnArgs& a, int mode, cudaStream_t s);

// ---- core.cu ----------------------------------------------------------------
void launch_factor_tables(const Geometry& g, int nterms, const double* term_weights,
                          const double* profiles, double* W0, double* W1, double* W2,
                          double* D, double* G, cudaStream_t s);
void launch_core_forward(const Geometry& g, int S, const double* T1, const double* W0,
                         const double* W1, double* T2, const double* colq, double* F,
                         cudaStream_t s);
void launch_core_backward(const Geometry& g, const double* G, const double* F,
                          double correction, const double* W0, const double* W1, double* B2,
                          double* corr_out, cudaStream_t s);
// F[e] = sum_b Fpart[b][e] over nblocks partial cores, blocks in order
void launch_core_sum(const Geometry& g, int nblocks, const double* Fpart, double* F,
                     cudaStream_t s);
// corr = correction * sum(colq), columns in order
void launch_charge_correction(const Geometry& g, int S, const double* colq, double correction,
                              double* corr, cudaStream_t s);
// WL[r][c L + a] = sum_i W[r][c L + i] Lam[i][a] for one axis
void launch_factor_wl(const Geometry& g, int axis, const double* W, const double* lam, double* WL,
                      cudaStream_t s);
void launch_axis_operands(const Geometry& g, int axis, int nterms, const double* W,
                          const double* D, double* out, cudaStream_t s);
// inverse == false: src = cells, dst = mesh; inverse == true: src = mesh, dst = cells
void launch_cells_to_mesh(const Geometry& g, const double* src, double* dst, bool inverse,
                          cudaStream_t s);

// ---- dense.cu ---------------------------------------------------------------
void dgemm_tn(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* in,
              const double* F, double* out, bool accumulate);
// batch entries z: in + z sin, F + z sF, out + z sout
void dgemm_tn_batched(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* in,
                      int64_t sin, const double* F, int64_t sF, double* out, int64_t sout,
                      int batch, bool accumulate);
size_t dense_workspace_bytes(int n0, int n1, int n2, int nterms);
// y[n0 n1][n2o] (+)= sum_r (A_r (x) B_r (x) C_r[:, coff : coff + nzi]) x[n0][n1][nzi]
// (C_r row-major [n2o][ldc]): the dense operator with a column slice of the
// last factor -- one z-slab's contribution to every output plane.
size_t kron_local_workspace_bytes(int n0, int n1, int nzi, int n2o, int nterms);
void kron_local(cudaStream_t s, int n0, int n1, int nzi, int n2o, int nterms, const double* A,
                const double* B, const double* C, int ldc, int coff, const double* x, double* y,
                bool accumulate, double* work, size_t work_bytes);
void kron_matvec_dense(cudaStream_t s, int n0, int n1, int n2, int nterms, const double* A,
                       const double* B, const double* C, const double* x, double* y,
                       double* work, size_t work_bytes);

}  // namespace kb
