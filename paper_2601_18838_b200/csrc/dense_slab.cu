// dense_slab.cu -- the dense SKP grid operator (config 5) on z-slabs of the
// mesh, one rank per GPU: y = sum_r (A_r (x) B_r (x) C_r) x with x and y
// distributed as slabs x_local[n0][n1][z_hi - z_lo] (rank order = z order).
//
// The reference applies the sharded axis through ordered axis-group
// all-reduces (spkmv, parallel.hpp:169-176). Three strategies for the
// non-local z product, all on the FP64 DMMA GEMM (dense.cu), the collectives
// over the plan's own NCCL communicator (one process per GPU) or, for a group
// of ranks held by one process, by peer copies in rank order:
//   REDUCE_SCATTER  every rank contracts its z-slice into full-length partial
//                   sums over all terms (the term-concatenated last pass,
//                   kron_local with a column slice of C_r), one reduce-scatter
//                   of the z-slabs -- the SPKMV pattern of the reference
//   RANK_SPLIT      all-gather the slabs, every rank applies its share of the
//                   terms (r = rank, rank + W, ...) to the whole mesh,
//                   reduce-scatter (the north star's rank split + reduce)
//   ALLTOALL        per term chunk, the x and y products on the z-slab, an
//                   all-to-all transpose to x-slabs, the term-concatenated z
//                   product, and one all-to-all back (the north star's slab
//                   all-to-all transpose)
// Slabs may be uneven; the block collectives pad every block to the largest
// slab. Every buffer is allocated once, at create.
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include <nccl.h>

#include "internal.h"

namespace kb {
extern thread_local std::string g_last_error;
}

using kb::Error;

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return KPME_GPU_OK;
    } catch (const Error& e) {
        kb::g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        kb::g_last_error = e.what();
        return KPME_GPU_RUNTIME;
    }
}

[[noreturn]] void invalid(const char* m) { throw Error(KPME_GPU_INVALID_ARGUMENT, m); }

#define DS_NCCL(call)                                                                         \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            throw Error(KPME_GPU_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));    \
    } while (0)

int split(int k, int i, int parts) { return (int)((int64_t)k * i / parts); }

// dst[s][m][0 : hi_s - lo_s] = src[m][lo_s : hi_s]: a [M][n2] array to slab-major
// blocks (block stride bs); inverse copies back.
__global__ void k_pack_slabs(int64_t M, int n2, int W, const int* __restrict__ lo,
                             const int* __restrict__ hi, int64_t bs, const double* __restrict__ src,
                             double* __restrict__ dst, int inverse) {
    const int64_t total = M * n2;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = e / n2;
        const int z = (int)(e % n2);
        int s = 0;
        while (s + 1 < W && z >= hi[s]) ++s;
        const int nz = hi[s] - lo[s];
        const int64_t d = (int64_t)s * bs + m * nz + (z - lo[s]);
        if (inverse)
            dst[e] = src[d];
        else
            dst[d] = src[e];
    }
}

// out[e] = sum_s part[s * bs + e], s ascending (fixed order).
__global__ void k_sum_blocks(int64_t n, int W, int64_t bs, const double* __restrict__ part,
                             double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < W; ++s) acc += part[(int64_t)s * bs + e];
        out[e] = acc;
    }
}

// send_q[r][z][x - xlo_q][y] = t2[r][z][x][y] for every destination q:
// the z-slab's x/y products split by destination x-slab (alltoall forward).
__global__ void k_pack_xslabs(int cr, int nz, int n0, int n1, int W, const int* __restrict__ xlo,
                              const int* __restrict__ xhi, const double* __restrict__ t2,
                              double* __restrict__ send) {
    const int64_t total = (int64_t)cr * nz * n0 * n1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(e % n1);
        const int x = (int)((e / n1) % n0);
        const int64_t rz = e / ((int64_t)n0 * n1);  // r * nz + z
        int q = 0;
        while (q + 1 < W && x >= xhi[q]) ++q;
        const int nx = xhi[q] - xlo[q];
        // block q starts at cr * nz * n1 * xlo[q]
        const int64_t d = (int64_t)cr * nz * n1 * xlo[q] + (rz * nx + (x - xlo[q])) * n1 + y;
        send[d] = t2[e];
    }
}

// Ccat[z'][k] over k = (q, r, z) with z < nz_q: C_{r0 + r}[z'][zlo_q + z]
// (the alltoall's last-pass operand; its row order matches the received
// blocks [q][r][z][(x, y)]).
__global__ void k_concat_qrz(int cr, int n2, int W, const int* __restrict__ zlo,
                             const int* __restrict__ zhi, const double* __restrict__ C,
                             double* __restrict__ Ccat) {
    const int64_t K = (int64_t)cr * n2;
    const int64_t total = (int64_t)n2 * K;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int zp = (int)(e / K);
        int64_t k = e % K;
        int q = 0;
        while (k >= (int64_t)cr * (zhi[q] - zlo[q])) {
            k -= (int64_t)cr * (zhi[q] - zlo[q]);
            ++q;
        }
        const int nz = zhi[q] - zlo[q];
        const int r = (int)(k / nz), z = (int)(k % nz);
        Ccat[e] = C[((int64_t)r * n2 + zp) * n2 + zlo[q] + z];
    }
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

}  // namespace

struct DsRank {
    int rank = 0, device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    const double *A = nullptr, *B = nullptr, *C = nullptr;  // [nt][n][n] on this device
    cudaEvent_t ev = nullptr;
    int* bounds = nullptr;  // device: zlo[W], zhi[W], xlo[W], xhi[W]
    double *ws = nullptr, *ypart = nullptr, *ysm = nullptr, *rsbuf = nullptr, *recv = nullptr;
    double *xsend = nullptr, *xall = nullptr, *xfull = nullptr;
    double *t1 = nullptr, *t2 = nullptr, *send = nullptr, *arecv = nullptr, *ccat = nullptr,
           *yx = nullptr;
    size_t ws_bytes = 0;
    std::vector<void*> allocs;
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        KB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

struct kpme_gpu_dense_slab_s {
    int n0 = 0, n1 = 0, n2 = 0, nt = 0, W = 1;
    bool group = false;        // every rank held by this process
    ncclComm_t comm = nullptr; // one rank per process
    std::vector<int> zlo, zhi, xlo, xhi;
    int maxnz = 0, maxnx = 0, chunk = 1;
    std::vector<DsRank> ranks;  // local ranks (1, or W for a group)
    ~kpme_gpu_dense_slab_s() {
        int prev = -1;
        cudaGetDevice(&prev);
        if (comm) ncclCommDestroy(comm);
        for (auto& r : ranks) {
            cudaSetDevice(r.device);
            if (r.ev) cudaEventDestroy(r.ev);
            if (r.own_stream && r.stream) cudaStreamDestroy(r.stream);
            for (void* p : r.allocs) cudaFree(p);
        }
        if (prev >= 0) cudaSetDevice(prev);
    }
    int64_t blk() const { return (int64_t)n0 * n1 * maxnz; }
};

namespace {

using DS = kpme_gpu_dense_slab_s;

void setup(DS* d) {
    const int W = d->W;
    for (int s = 0; s < W; ++s) {
        d->zlo.push_back(split(d->n2, s, W));
        d->zhi.push_back(split(d->n2, s + 1, W));
        d->xlo.push_back(split(d->n0, s, W));
        d->xhi.push_back(split(d->n0, s + 1, W));
        d->maxnz = std::max(d->maxnz, d->zhi[s] - d->zlo[s]);
        d->maxnx = std::max(d->maxnx, d->xhi[s] - d->xlo[s]);
    }
    d->chunk = std::max(1, std::min(d->nt, 8));
    const int64_t mesh = (int64_t)d->n0 * d->n1 * d->n2;
    for (auto& r : d->ranks) {
        const kb::DeviceGuard dg(r.device);
        KB_CUDA(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
        r.own_stream = true;
        KB_CUDA(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
        std::vector<int> b;
        for (auto* v : {&d->zlo, &d->zhi, &d->xlo, &d->xhi}) b.insert(b.end(), v->begin(), v->end());
        r.bounds = r.alloc<int>(b.size());
        KB_CUDA(cudaMemcpy(r.bounds, b.data(), sizeof(int) * b.size(), cudaMemcpyHostToDevice));
        const int nz = d->zhi[r.rank] - d->zlo[r.rank];
        // rank_split applies its terms one kron_local call each (strided operands)
        r.ws_bytes = std::max(kb::kron_local_workspace_bytes(d->n0, d->n1, nz, d->n2, d->nt),
                              kb::kron_local_workspace_bytes(d->n0, d->n1, d->n2, d->n2, 1));
        r.ws = r.alloc<double>(r.ws_bytes / sizeof(double) + 1);
        r.ypart = r.alloc<double>(mesh);
        r.ysm = r.alloc<double>((size_t)W * d->blk());
        r.recv = r.alloc<double>(d->blk());
        if (d->group) r.rsbuf = r.alloc<double>((size_t)W * d->blk());
        r.xsend = r.alloc<double>(d->blk());
        r.xall = r.alloc<double>((size_t)W * d->blk());
        r.xfull = r.alloc<double>(mesh);
        const int64_t cm = (int64_t)d->chunk * d->n0 * d->n1 * nz;
        r.t1 = r.alloc<double>(cm);
        r.t2 = r.alloc<double>(cm);
        r.send = r.alloc<double>(std::max<int64_t>(cm, (int64_t)W * d->maxnx * d->n1 * d->maxnz));
        r.arecv = r.alloc<double>(std::max<int64_t>((int64_t)d->chunk * d->maxnx * d->n1 * d->n2,
                                                    (int64_t)d->n0 * d->n1 * d->maxnz));
        r.ccat = r.alloc<double>((int64_t)d->n2 * d->chunk * d->n2);
        r.yx = r.alloc<double>((int64_t)d->maxnx * d->n1 * d->n2);
    }
}

// Every local stream waits for every other (before / after group copies).
void barrier(DS* d) {
    if (d->ranks.size() < 2) return;
    for (auto& r : d->ranks) {
        const kb::DeviceGuard dg(r.device);
        KB_CUDA(cudaEventRecord(r.ev, r.stream));
    }
    for (auto& r : d->ranks) {
        const kb::DeviceGuard dg(r.device);
        for (auto& o : d->ranks)
            if (&o != &r) KB_CUDA(cudaStreamWaitEvent(r.stream, o.ev, 0));
    }
}

// All-gather of one padded block per rank: xall[s] = xsend of rank s.
void allgather(DS* d) {
    const int64_t bs = d->blk();
    if (!d->group) {
        DsRank& r = d->ranks[0];
        if (d->W == 1) {
            KB_CUDA(cudaMemcpyAsync(r.xall, r.xsend, sizeof(double) * bs, cudaMemcpyDeviceToDevice,
                                    r.stream));
            return;
        }
        const kb::DeviceGuard dg(r.device);
        DS_NCCL(ncclAllGather(r.xsend, r.xall, bs, ncclDouble, d->comm, r.stream));
        return;
    }
    barrier(d);
    for (auto& dst : d->ranks) {
        const kb::DeviceGuard dg(dst.device);
        for (auto& src : d->ranks)
            KB_CUDA(cudaMemcpyPeerAsync(dst.xall + src.rank * bs, dst.device, src.xsend, src.device,
                                        sizeof(double) * bs, dst.stream));
    }
    barrier(d);
}

// Reduce-scatter of W padded blocks: recv = sum_s ysm_s[rank], s ascending.
void reduce_scatter(DS* d) {
    const int64_t bs = d->blk();
    if (!d->group) {
        DsRank& r = d->ranks[0];
        const kb::DeviceGuard dg(r.device);
        if (d->W == 1) {
            KB_CUDA(cudaMemcpyAsync(r.recv, r.ysm, sizeof(double) * bs, cudaMemcpyDeviceToDevice,
                                    r.stream));
            return;
        }
        DS_NCCL(ncclReduceScatter(r.ysm, r.recv, bs, ncclDouble, ncclSum, d->comm, r.stream));
        return;
    }
    barrier(d);
    for (auto& dst : d->ranks) {
        const kb::DeviceGuard dg(dst.device);
        for (auto& src : d->ranks)
            KB_CUDA(cudaMemcpyPeerAsync(dst.rsbuf + src.rank * bs, dst.device,
                                        src.ysm + dst.rank * bs, src.device, sizeof(double) * bs,
                                        dst.stream));
        k_sum_blocks<<<grid_for(bs), 256, 0, dst.stream>>>(bs, d->W, bs, dst.rsbuf, dst.recv);
        KB_CHECK_LAUNCH();
    }
    barrier(d);
}

// All-to-all with per-pair counts: rank d receives, in source order, cnt(s, d)
// doubles from offset soff(s, d) of rank s's `sendbuf` at roff(d, s) of its
// `recvbuf`.
template <class Cnt, class Soff, class Roff>
void alltoallv(DS* d, double* DsRank::*sendbuf, double* DsRank::*recvbuf, Cnt cnt, Soff soff,
               Roff roff) {
    if (!d->group) {
        DsRank& r = d->ranks[0];
        const kb::DeviceGuard dg(r.device);
        if (d->W == 1) {
            const int64_t c = cnt(0, 0);
            if (c > 0)
                KB_CUDA(cudaMemcpyAsync(r.*recvbuf + roff(0, 0), r.*sendbuf + soff(0, 0),
                                        sizeof(double) * c, cudaMemcpyDeviceToDevice, r.stream));
            return;
        }
        DS_NCCL(ncclGroupStart());
        for (int q = 0; q < d->W; ++q) {
            const int64_t cs = cnt(r.rank, q), cr = cnt(q, r.rank);
            if (cs > 0) DS_NCCL(ncclSend(r.*sendbuf + soff(r.rank, q), cs, ncclDouble, q, d->comm, r.stream));
            if (cr > 0) DS_NCCL(ncclRecv(r.*recvbuf + roff(r.rank, q), cr, ncclDouble, q, d->comm, r.stream));
        }
        DS_NCCL(ncclGroupEnd());
        return;
    }
    barrier(d);
    for (auto& dst : d->ranks) {
        const kb::DeviceGuard dg(dst.device);
        for (auto& src : d->ranks) {
            const int64_t c = cnt(src.rank, dst.rank);
            if (c > 0)
                KB_CUDA(cudaMemcpyPeerAsync(dst.*recvbuf + roff(dst.rank, src.rank), dst.device,
                                            src.*sendbuf + soff(src.rank, dst.rank), src.device,
                                            sizeof(double) * c, dst.stream));
        }
    }
    barrier(d);
}

void apply_reduce_scatter(DS* d, const double* const* x, double* const* y) {
    const int64_t M = (int64_t)d->n0 * d->n1;
    for (size_t i = 0; i < d->ranks.size(); ++i) {
        DsRank& r = d->ranks[i];
        const kb::DeviceGuard dg(r.device);
        const int nz = d->zhi[r.rank] - d->zlo[r.rank];
        kb::kron_local(r.stream, d->n0, d->n1, nz, d->n2, d->nt, r.A, r.B, r.C, d->n2,
                       d->zlo[r.rank], x[i], r.ypart, false, r.ws, r.ws_bytes);
        k_pack_slabs<<<grid_for(M * d->n2), 256, 0, r.stream>>>(M, d->n2, d->W, r.bounds,
                                                               r.bounds + d->W, d->blk(), r.ypart,
                                                               r.ysm, 0);
        KB_CHECK_LAUNCH();
    }
    reduce_scatter(d);
    for (size_t i = 0; i < d->ranks.size(); ++i) {
        DsRank& r = d->ranks[i];
        const kb::DeviceGuard dg(r.device);
        const int nz = d->zhi[r.rank] - d->zlo[r.rank];
        KB_CUDA(cudaMemcpyAsync(y[i], r.recv, sizeof(double) * M * nz, cudaMemcpyDeviceToDevice,
                                r.stream));
    }
}

void apply_rank_split(DS* d, const double* const* x, double* const* y) {
    const int64_t M = (int64_t)d->n0 * d->n1;
    for (size_t i = 0; i < d->ranks.size(); ++i) {
        DsRank& r = d->ranks[i];
        const kb::DeviceGuard dg(r.device);
        const int nz = d->zhi[r.rank] - d->zlo[r.rank];
        KB_CUDA(cudaMemcpyAsync(r.xsend, x[i], sizeof(double) * M * nz, cudaMemcpyDeviceToDevice,
                                r.stream));
    }
    allgather(d);
    for (size_t i = 0; i < d->ranks.size(); ++i) {
        DsRank& r = d->ranks[i];
        const kb::DeviceGuard dg(r.device);
        k_pack_slabs<<<grid_for(M * d->n2), 256, 0, r.stream>>>(M, d->n2, d->W, r.bounds,
                                                               r.bounds + d->W, d->blk(), r.xall,
                                                               r.xfull, 1);
        KB_CHECK_LAUNCH();
        // terms rank, rank + W, ...: strided operands, one kron_local per term
        bool first = true;
        for (int t = r.rank; t < d->nt; t += d->W) {
            const int64_t s0 = (int64_t)d->n0 * d->n0, s1 = (int64_t)d->n1 * d->n1,
                          s2 = (int64_t)d->n2 * d->n2;
            kb::kron_local(r.stream, d->n0, d->n1, d->n2, d->n2, 1, r.A + t * s0, r.B + t * s1,
                           r.C + t * s2, d->n2, 0, r.xfull, r.ypart, !first, r.ws, r.ws_bytes);
            first = false;
        }
        if (first) KB_CUDA(cudaMemsetAsync(r.ypart, 0, sizeof(double) * M * d->n2, r.stream));
        k_pack_slabs<<<grid_for(M * d->n2), 256, 0, r.stream>>>(M, d->n2, d->W, r.bounds,
                                                               r.bounds + d->W, d->blk(), r.ypart,
                                                               r.ysm, 0);
        KB_CHECK_LAUNCH();
    }
    reduce_scatter(d);
    for (size_t i = 0; i < d->ranks.size(); ++i) {
        DsRank& r = d->ranks[i];
        const kb::DeviceGuard dg(r.device);
        const int nz = d->zhi[r.rank] - d->zlo[r.rank];
        KB_CUDA(cudaMemcpyAsync(y[i], r.recv, sizeof(double) * M * nz, cudaMemcpyDeviceToDevice,
                                r.stream));
    }
}

void apply_alltoall(DS* d, const double* const* x, double* const* y) {
    const int W = d->W, n0 = d->n0, n1 = d->n1, n2 = d->n2;
    auto nzs = [&](int s) { return d->zhi[s] - d->zlo[s]; };
    auto nxs = [&](int s) { return d->xhi[s] - d->xlo[s]; };
    for (auto& r : d->ranks) {
        const kb::DeviceGuard dg(r.device);
        KB_CUDA(cudaMemsetAsync(r.yx, 0, sizeof(double) * nxs(r.rank) * n1 * n2, r.stream));
    }
    for (int r0 = 0; r0 < d->nt; r0 += d->chunk) {
        const int cr = std::min(d->chunk, d->nt - r0);
        for (size_t i = 0; i < d->ranks.size(); ++i) {
            DsRank& r = d->ranks[i];
            const kb::DeviceGuard dg(r.device);
            const int nz = nzs(r.rank);
            const int64_t mi = (int64_t)n0 * n1 * nz;
            if (nz == 0) continue;
            kb::dgemm_tn_batched(r.stream, (int64_t)n1 * nz, n0, n0, x[i], 0,
                                 r.A + (int64_t)r0 * n0 * n0, (int64_t)n0 * n0, r.t1, mi, cr, false);
            kb::dgemm_tn_batched(r.stream, (int64_t)nz * n0, n1, n1, r.t1, mi,
                                 r.B + (int64_t)r0 * n1 * n1, (int64_t)n1 * n1, r.t2, mi, cr, false);
            k_pack_xslabs<<<grid_for(cr * mi), 256, 0, r.stream>>>(cr, nz, n0, n1, W,
                                                                  r.bounds + 2 * W, r.bounds + 3 * W,
                                                                  r.t2, r.send);
            KB_CHECK_LAUNCH();
        }
        // rank s sends [r][z_s][x_q][y] to rank q; q stores it at block s
        alltoallv(
            d, &DsRank::send, &DsRank::arecv,
            [&](int s, int q) { return (int64_t)cr * nzs(s) * nxs(q) * n1; },
            [&](int s, int q) { return (int64_t)cr * nzs(s) * n1 * d->xlo[q]; },
            [&](int q, int s) { return (int64_t)cr * n1 * nxs(q) * d->zlo[s]; });
        for (auto& r : d->ranks) {
            const kb::DeviceGuard dg(r.device);
            const int nx = nxs(r.rank);
            k_concat_qrz<<<grid_for((int64_t)n2 * cr * n2), 256, 0, r.stream>>>(
                cr, n2, W, r.bounds, r.bounds + W, r.C + (int64_t)r0 * n2 * n2, r.ccat);
            KB_CHECK_LAUNCH();
            if (nx > 0)
                kb::dgemm_tn(r.stream, (int64_t)nx * n1, n2, (int64_t)cr * n2, r.arecv, r.ccat,
                             r.yx, true);
        }
    }
    // back to z-slabs: rank s sends yx[x_s][y][zlo_q : zhi_q] to q, which
    // stores it at x offset xlo_s: y_local = [n0][n1][nz_q]
    for (auto& r : d->ranks) {
        const kb::DeviceGuard dg(r.device);
        const int64_t M = (int64_t)nxs(r.rank) * n1;
        if (M > 0) {
            k_pack_slabs<<<grid_for(M * n2), 256, 0, r.stream>>>(M, n2, W, r.bounds, r.bounds + W,
                                                                (int64_t)d->maxnx * n1 * d->maxnz,
                                                                r.yx, r.send, 0);
            KB_CHECK_LAUNCH();
        }
    }
    alltoallv(
        d, &DsRank::send, &DsRank::arecv,
        [&](int s, int q) { return (int64_t)nxs(s) * n1 * nzs(q); },
        [&](int s, int q) { return (int64_t)q * d->maxnx * n1 * d->maxnz; },
        [&](int q, int s) { return (int64_t)d->xlo[s] * n1 * nzs(q); });
    for (size_t i = 0; i < d->ranks.size(); ++i) {
        DsRank& r = d->ranks[i];
        const kb::DeviceGuard dg(r.device);
        KB_CUDA(cudaMemcpyAsync(y[i], r.arecv, sizeof(double) * n0 * n1 * nzs(r.rank),
                                cudaMemcpyDeviceToDevice, r.stream));
    }
}

void apply(DS* d, int strategy, const double* const* x, double* const* y) {
    if (!x || !y) invalid("kpme_gpu_dense_slab_apply: null slab arrays");
    switch (strategy) {
        case KPME_GPU_SLAB_REDUCE_SCATTER: return apply_reduce_scatter(d, x, y);
        case KPME_GPU_SLAB_RANK_SPLIT: return apply_rank_split(d, x, y);
        case KPME_GPU_SLAB_ALLTOALL: return apply_alltoall(d, x, y);
        default: invalid("kpme_gpu_dense_slab_apply: unknown strategy");
    }
}

void check_shape(int n0, int n1, int n2, int nterms, int W) {
    if (n0 < 1 || n1 < 1 || n2 < 1 || nterms < 0) invalid("kpme_gpu_dense_slab: bad shape");
    if (W < 1 || W > kb::PerDevice::kMax) invalid("kpme_gpu_dense_slab: bad rank count");
    if (W > n2 || W > n0) invalid("kpme_gpu_dense_slab: more ranks than mesh planes");
}

}  // namespace

extern "C" int kpme_gpu_dense_slab_create(int device, int n0, int n1, int n2, int nterms,
                                          const double* A, const double* B, const double* C,
                                          int nranks, int rank, const void* nccl_id,
                                          kpme_gpu_dense_slab* out) {
    return guarded([&] {
        check_shape(n0, n1, n2, nterms, nranks);
        if (!out || !A || !B || !C) invalid("kpme_gpu_dense_slab_create: null argument");
        if (rank < 0 || rank >= nranks) invalid("kpme_gpu_dense_slab_create: bad rank");
        if (nranks > 1 && !nccl_id) invalid("kpme_gpu_dense_slab_create: NCCL id required");
        const kb::DeviceGuard dg(device);
        auto d = new DS();
        try {
            d->n0 = n0, d->n1 = n1, d->n2 = n2, d->nt = nterms, d->W = nranks;
            DsRank r;
            r.rank = rank, r.device = device, r.A = A, r.B = B, r.C = C;
            d->ranks.push_back(r);
            setup(d);
            if (nranks > 1) {
                ncclUniqueId u;
                std::memcpy(&u, nccl_id, sizeof(u));
                DS_NCCL(ncclCommInitRank(&d->comm, nranks, u, rank));
            }
            *out = d;
        } catch (...) {
            delete d;
            throw;
        }
    });
}

extern "C" int kpme_gpu_dense_slab_create_group(int nranks, const int* devices, int n0, int n1,
                                                int n2, int nterms, const double* const* A,
                                                const double* const* B, const double* const* C,
                                                kpme_gpu_dense_slab* out) {
    return guarded([&] {
        check_shape(n0, n1, n2, nterms, nranks);
        if (!out || !devices || !A || !B || !C) invalid("kpme_gpu_dense_slab_create_group: null argument");
        auto d = new DS();
        try {
            d->n0 = n0, d->n1 = n1, d->n2 = n2, d->nt = nterms, d->W = nranks;
            d->group = true;
            for (int s = 0; s < nranks; ++s) {
                DsRank r;
                r.rank = s, r.device = devices[s], r.A = A[s], r.B = B[s], r.C = C[s];
                d->ranks.push_back(r);
            }
            for (int i = 0; i < nranks; ++i)
                for (int j = 0; j < nranks; ++j) {
                    const int di = devices[i], dj = devices[j];
                    if (di == dj) continue;
                    const kb::DeviceGuard dg(di);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled || e == cudaErrorPeerAccessUnsupported)
                        cudaGetLastError();  // copies still work (staged) without peer access
                    else if (e != cudaSuccess)
                        KB_CUDA(e);
                }
            setup(d);
            *out = d;
        } catch (...) {
            delete d;
            throw;
        }
    });
}

extern "C" int kpme_gpu_dense_slab_destroy(kpme_gpu_dense_slab h) {
    return guarded([&] { delete h; });
}

extern "C" int kpme_gpu_dense_slab_bounds(kpme_gpu_dense_slab h, int rank, int* z_lo, int* z_hi) {
    return guarded([&] {
        if (!h || rank < 0 || rank >= h->W || !z_lo || !z_hi) invalid("kpme_gpu_dense_slab_bounds: bad argument");
        *z_lo = h->zlo[rank];
        *z_hi = h->zhi[rank];
    });
}

extern "C" int kpme_gpu_dense_slab_set_stream(kpme_gpu_dense_slab h, int local, void* stream) {
    return guarded([&] {
        if (!h || local < 0 || local >= (int)h->ranks.size()) invalid("kpme_gpu_dense_slab_set_stream: bad rank");
        DsRank& r = h->ranks[local];
        const kb::DeviceGuard dg(r.device);
        if (r.own_stream && r.stream) KB_CUDA(cudaStreamDestroy(r.stream));
        r.own_stream = false;
        r.stream = static_cast<cudaStream_t>(stream);
    });
}

extern "C" int kpme_gpu_dense_slab_apply(kpme_gpu_dense_slab h, int strategy,
                                         const double* const* x_local, double* const* y_local) {
    return guarded([&] {
        if (!h) invalid("kpme_gpu_dense_slab_apply: null handle");
        apply(h, strategy, x_local, y_local);
    });
}

extern "C" int kpme_gpu_dense_slab_sync(kpme_gpu_dense_slab h) {
    return guarded([&] {
        if (!h) invalid("kpme_gpu_dense_slab_sync: null handle");
        for (auto& r : h->ranks) {
            const kb::DeviceGuard dg(r.device);
            KB_CUDA(cudaStreamSynchronize(r.stream));
        }
    });
}

extern "C" int kpme_gpu_dense_slab_choose(kpme_gpu_dense_slab h, const double* const* x_local,
                                          double* const* y_local, int reps, double* ms,
                                          int* best) {
    return guarded([&] {
        if (!h || !ms || !best) invalid("kpme_gpu_dense_slab_choose: null argument");
        reps = std::max(1, reps);
        DsRank& r0 = h->ranks[0];
        double* dmax = nullptr;
        for (int s = 0; s < 3; ++s) {
            apply(h, s, x_local, y_local);  // warm
            barrier(h);
            cudaEvent_t e0, e1;
            const kb::DeviceGuard dg(r0.device);
            KB_CUDA(cudaEventCreate(&e0));
            KB_CUDA(cudaEventCreate(&e1));
            KB_CUDA(cudaEventRecord(e0, r0.stream));
            for (int k = 0; k < reps; ++k) apply(h, s, x_local, y_local);
            barrier(h);
            KB_CUDA(cudaEventRecord(e1, r0.stream));
            KB_CUDA(cudaEventSynchronize(e1));
            float t = 0.f;
            KB_CUDA(cudaEventElapsedTime(&t, e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            double v = t / reps;
            if (h->comm && h->W > 1) {  // max over ranks
                if (!dmax) KB_CUDA(cudaMalloc(&dmax, sizeof(double)));
                KB_CUDA(cudaMemcpyAsync(dmax, &v, sizeof(double), cudaMemcpyHostToDevice, r0.stream));
                DS_NCCL(ncclAllReduce(dmax, dmax, 1, ncclDouble, ncclMax, h->comm, r0.stream));
                KB_CUDA(cudaMemcpyAsync(&v, dmax, sizeof(double), cudaMemcpyDeviceToHost, r0.stream));
                KB_CUDA(cudaStreamSynchronize(r0.stream));
            }
            ms[s] = v;
        }
        if (dmax) cudaFree(dmax);
        *best = (int)(std::min_element(ms, ms + 3) - ms);
    });
}
