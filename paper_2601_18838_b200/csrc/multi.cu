// multi.cu -- multi-device plans: one host thread drives G devices.
//
// The reference runs kpme_apply over a K0 x K1 x K2 rank grid whose ranks
// exchange through ordered axis-group all-reduces (SimulatedComm,
// parallel.hpp:98-145; spkmv, parallel.hpp:156-179). A multi-device plan is
// that decomposition on one node: a P0 x P1 x P2 grid of cell blocks, one per
// device entry, ranks flattened like cells (RankGrid, parallel.hpp:46-82).
//
//   every device   route: keep its block's particles, in ascending index order
//                  (stable compaction; the out-of-box check of
//                  assign_particles, geometry.hpp:136-138, on the way)
//                  sort -> spread -> forward contractions -> partial core
//   exchange       the collapsed form's only collective: sum of the G partial
//                  R^3 + 1 cores (the last entry carries sum q). PEER: every
//                  device sums all G cores itself, in rank order, straight
//                  from its peers' memory over NVLink (no NCCL round, same
//                  bits on every device); NCCL: one grouped ncclAllReduce.
//   every device   backward expansions -> gather of its particles
//   home device    peers' potentials arrive by peer copy and are scattered
//                  to global particle order (KpmeResult::potentials).
//
// A device may appear more than once in the list (several blocks on one
// GPU): the PEER path then reads local memory, which is how the decomposition
// is tested on a single B200.
#include <algorithm>
#include <climits>
#include <cstring>

#include "plan.h"

namespace kb {

namespace {

constexpr int kRouteThreads = 256;
constexpr int kRoutePer = 8;  // consecutive particles per thread
constexpr int kRouteTile = kRouteThreads * kRoutePer;

__device__ __forceinline__ bool in_block(const Geometry& g, double p0, double p1, double p2,
                                         int64_t i, unsigned long long* bad) {
    if (fabs(p0 - g.center[0]) > g.radius || fabs(p1 - g.center[1]) > g.radius ||
        fabs(p2 - g.center[2]) > g.radius)
        atomicMin(bad, (unsigned long long)i);  // Box3::contains, geometry.hpp:36-40
    const double b = __dmul_rn(2.0, g.radius), y = g.inv_diam;
    const int c0 = exact_axis_cell(p0, g.center[0], g.radius, g.K[0], b, y);
    const int c1 = exact_axis_cell(p1, g.center[1], g.radius, g.K[1], b, y);
    const int c2 = exact_axis_cell(p2, g.center[2], g.radius, g.K[2], b, y);
    return c0 >= g.x_lo && c0 < g.x_hi && c1 >= g.y_lo && c1 < g.y_hi && c2 >= g.z_lo &&
           c2 < g.z_hi;
}

// Block-wide exclusive scan of one int per thread (256 threads).
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
    __shared__ int wsum[kRouteThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < kRouteThreads / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kRouteThreads / 32) wsum[lane] = s;
    }
    __syncthreads();
    const int base = w ? wsum[w - 1] : 0;
    *total = wsum[kRouteThreads / 32 - 1];
    __syncthreads();
    return base + x - v;
}

// Pass 1: particles of the block per tile of 2048 (thread t owns particles
// tile*2048 + 8t .. 8t+7).
__global__ void __launch_bounds__(kRouteThreads) k_route_count(Geometry g, int64_t n,
                                                               const double* __restrict__ xyz,
                                                               int32_t* __restrict__ tiles,
                                                               unsigned long long* bad) {
    const int64_t i0 = (int64_t)blockIdx.x * kRouteTile + (int64_t)threadIdx.x * kRoutePer;
    int c = 0;
    for (int k = 0; k < kRoutePer; ++k) {
        const int64_t i = i0 + k;
        if (i < n) c += in_block(g, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], i, bad) ? 1 : 0;
    }
    int total;
    block_excl_scan(c, &total);
    if (threadIdx.x == 0) tiles[blockIdx.x] = total;
}

// Pass 2: stable scatter. Each CTA sums the counts of the tiles before it
// (at most a few thousand), then every thread writes its block particles in
// index order; the last CTA writes the total.
__global__ void __launch_bounds__(kRouteThreads) k_route_scatter(
    Geometry g, int64_t n, const double* __restrict__ xyz, const double* __restrict__ q,
    const int32_t* __restrict__ tiles, double* __restrict__ xyz_c, double* __restrict__ q_c,
    int32_t* __restrict__ idx, int64_t* count, unsigned long long* bad) {
    int pre = 0;
    for (int t = threadIdx.x; t < (int)blockIdx.x; t += kRouteThreads) pre += tiles[t];
    int tot_pre;
    block_excl_scan(pre, &tot_pre);
    const int64_t i0 = (int64_t)blockIdx.x * kRouteTile + (int64_t)threadIdx.x * kRoutePer;
    unsigned keep = 0;
    int c = 0;
    for (int k = 0; k < kRoutePer; ++k) {
        const int64_t i = i0 + k;
        if (i < n && in_block(g, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], i, bad)) {
            keep |= 1u << k;
            ++c;
        }
    }
    int total;
    int64_t pos = (int64_t)tot_pre + block_excl_scan(c, &total);
    for (int k = 0; k < kRoutePer; ++k) {
        if (!(keep >> k & 1u)) continue;
        const int64_t i = i0 + k;
        xyz_c[3 * pos] = xyz[3 * i];
        xyz_c[3 * pos + 1] = xyz[3 * i + 1];
        xyz_c[3 * pos + 2] = xyz[3 * i + 2];
        q_c[pos] = q[i];
        idx[pos] = (int32_t)i;
        ++pos;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *count = (int64_t)tot_pre + total;
}

// Fixed-order sum of G partial cores, read where they live (local or peer
// memory): out[e] = sum_{d ascending} cores[d][e].
__global__ void k_sum_cores(const double* const* __restrict__ cores, int G, int E,
                            double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int d = 0; d < G; ++d) s += cores[d][e];
        out[e] = s;
    }
}

// out[idx[i]] = pot[i]: compacted potentials back to global particle order.
__global__ void k_scatter_out(int64_t n, const double* __restrict__ pot,
                              const int32_t* __restrict__ idx, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[idx[i]] = pot[i];
}

#define KB_NCCL(call)                                                                        \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess)                                                               \
            throw ::kb::Error(KPME_GPU_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

}  // namespace

struct Part {
    int device = 0;
    kpme_gpu_plan plan = nullptr;   // block plan on `device`
    double* xyz = nullptr;          // [cap][3] every particle (broadcast copy)
    double* q = nullptr;            // [cap]
    double* xyz_c = nullptr;        // [cap][3] the block's particles, ascending index
    double* q_c = nullptr;          // [cap]
    int32_t* idx = nullptr;         // [cap] their global indices
    int32_t* tiles = nullptr;       // [route tiles]
    int64_t* count_d = nullptr;     // [1]
    unsigned long long* bad = nullptr;  // [1] lowest out-of-box index
    double* core = nullptr;         // [E] partial core
    double* core_sum = nullptr;     // [E] summed core
    const double** core_ptrs = nullptr;  // [G] every part's partial core (device array)
    double* pot = nullptr;          // [cap] potentials of the block's particles
    cudaEvent_t ev_route = nullptr, ev_fwd = nullptr, ev_bwd = nullptr;
    int64_t count = 0;
    std::vector<void*> allocs;

    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        KB_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

struct MultiPlan {
    int dims[3] = {1, 1, 1};
    int G = 0;
    int coll = KPME_GPU_COLL_PEER;
    bool peer_ok = false;   // every device pair can reach each other's memory
    bool distinct = false;  // no device repeats (NCCL needs one rank per device)
    int64_t cap = 0;
    int E = 0;
    std::vector<Part> parts;
    std::vector<ncclComm_t> comms;
    // home device (parts[0].device): merge buffers
    double* pot_all = nullptr;
    int32_t* idx_all = nullptr;
    double* out_home = nullptr;
    int64_t* counts_h = nullptr;            // pinned [G]
    unsigned long long* bad_h = nullptr;    // pinned [G]
    std::vector<void*> home_allocs;
};

void destroy_multi(MultiPlan* m) {
    if (!m) return;
    int prev = -1;
    cudaGetDevice(&prev);
    for (auto c : m->comms)
        if (c) ncclCommDestroy(c);
    for (auto& pt : m->parts) {
        cudaSetDevice(pt.device);
        if (pt.ev_route) cudaEventDestroy(pt.ev_route);
        if (pt.ev_fwd) cudaEventDestroy(pt.ev_fwd);
        if (pt.ev_bwd) cudaEventDestroy(pt.ev_bwd);
        for (void* p : pt.allocs) cudaFree(p);
        if (pt.plan) kpme_gpu_plan_destroy(pt.plan);
    }
    if (!m->parts.empty()) {
        cudaSetDevice(m->parts[0].device);
        for (void* p : m->home_allocs) cudaFree(p);
    }
    if (m->counts_h) cudaFreeHost(m->counts_h);
    if (m->bad_h) cudaFreeHost(m->bad_h);
    if (prev >= 0) cudaSetDevice(prev);
    delete m;
}

}  // namespace kb

namespace kbp {

using kb::MultiPlan;
using kb::Part;

namespace {

void init_nccl(MultiPlan* m) {
    if (!m->comms.empty()) return;
    if (!m->distinct)
        invalid("kpme_gpu: the NCCL exchange needs distinct devices (one rank per GPU)");
    std::vector<int> devs;
    for (auto& pt : m->parts) devs.push_back(pt.device);
    m->comms.assign(m->G, nullptr);
    KB_NCCL(ncclCommInitAll(m->comms.data(), m->G, devs.data()));
}

// Broadcast (already done by the caller into part.xyz/q or given directly),
// route, and read the counts back: the block sizes set the launch shapes of
// everything after.
void route_all(MultiPlan* m, int64_t n, const double* const* xyz_of, const double* const* q_of) {
    const int ntiles = (int)std::max<int64_t>(1, (n + kb::kRouteTile - 1) / kb::kRouteTile);
    for (int d = 0; d < m->G; ++d) {
        Part& pt = m->parts[d];
        const kb::DeviceGuard dg(pt.device);
        cudaStream_t s = pt.plan->stream;
        KB_CUDA(cudaMemsetAsync(pt.bad, 0xff, sizeof(unsigned long long), s));
        KB_CUDA(cudaMemsetAsync(pt.count_d, 0, sizeof(int64_t), s));
        if (n > 0) {
            kb::k_route_count<<<ntiles, kb::kRouteThreads, 0, s>>>(pt.plan->g, n, xyz_of[d],
                                                                  pt.tiles, pt.bad);
            KB_CHECK_LAUNCH();
            kb::k_route_scatter<<<ntiles, kb::kRouteThreads, 0, s>>>(
                pt.plan->g, n, xyz_of[d], q_of[d], pt.tiles, pt.xyz_c, pt.q_c, pt.idx, pt.count_d,
                pt.bad);
            KB_CHECK_LAUNCH();
        }
        KB_CUDA(cudaMemcpyAsync(m->counts_h + d, pt.count_d, sizeof(int64_t),
                                cudaMemcpyDeviceToHost, s));
        KB_CUDA(cudaMemcpyAsync(m->bad_h + d, pt.bad, sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, s));
        KB_CUDA(cudaEventRecord(pt.ev_route, s));
    }
    for (int d = 0; d < m->G; ++d) KB_CUDA(cudaEventSynchronize(m->parts[d].ev_route));
    unsigned long long first = ULLONG_MAX;
    for (int d = 0; d < m->G; ++d) first = std::min(first, m->bad_h[d]);
    if (first != ULLONG_MAX)
        throw kb::Error(KPME_GPU_INVALID_ARGUMENT,
                        "assign_particles: particle " + std::to_string(first) + " outside the box");
    int64_t tot = 0;
    for (int d = 0; d < m->G; ++d) {
        m->parts[d].count = m->counts_h[d];
        tot += m->counts_h[d];
    }
    if (tot != n) throw kb::Error(KPME_GPU_RUNTIME, "kpme_gpu: cell blocks do not cover the box");
}

// forward halves, core exchange, backward halves; then peers' potentials are
// scattered to global order into `out` (home device memory).
void compute_and_merge(MultiPlan* m, int64_t n, double* out) {
    const int G = m->G;
    for (int d = 0; d < G; ++d) {
        Part& pt = m->parts[d];
        const kb::DeviceGuard dg(pt.device);
        forward_half(pt.plan, pt.count, pt.xyz_c, pt.q_c, pt.core);
        KB_CUDA(cudaEventRecord(pt.ev_fwd, pt.plan->stream));
    }
    if (m->coll == KPME_GPU_COLL_NCCL) {
        init_nccl(m);
        KB_NCCL(ncclGroupStart());
        for (int d = 0; d < G; ++d) {
            Part& pt = m->parts[d];
            const kb::DeviceGuard dg(pt.device);
            KB_NCCL(ncclAllReduce(pt.core, pt.core_sum, m->E, ncclDouble, ncclSum, m->comms[d],
                                  pt.plan->stream));
        }
        KB_NCCL(ncclGroupEnd());
    } else {
        for (int d = 0; d < G; ++d) {
            Part& pt = m->parts[d];
            const kb::DeviceGuard dg(pt.device);
            for (int e = 0; e < G; ++e)
                if (e != d) KB_CUDA(cudaStreamWaitEvent(pt.plan->stream, m->parts[e].ev_fwd, 0));
            kb::k_sum_cores<<<(m->E + 255) / 256, 256, 0, pt.plan->stream>>>(pt.core_ptrs, G, m->E,
                                                                             pt.core_sum);
            KB_CHECK_LAUNCH();
        }
    }
    for (int d = 0; d < G; ++d) {
        Part& pt = m->parts[d];
        const kb::DeviceGuard dg(pt.device);
        backward_half(pt.plan, pt.core_sum, pt.pot);
        KB_CUDA(cudaEventRecord(pt.ev_bwd, pt.plan->stream));
    }
    Part& home = m->parts[0];
    const kb::DeviceGuard dg(home.device);
    cudaStream_t hs = home.plan->stream;
    int64_t off = 0;
    for (int d = 0; d < G; ++d) {
        Part& pt = m->parts[d];
        if (d) KB_CUDA(cudaStreamWaitEvent(hs, pt.ev_bwd, 0));
        if (pt.count > 0) {
            KB_CUDA(cudaMemcpyPeerAsync(m->pot_all + off, home.device, pt.pot, pt.device,
                                        sizeof(double) * pt.count, hs));
            KB_CUDA(cudaMemcpyPeerAsync(m->idx_all + off, home.device, pt.idx, pt.device,
                                        sizeof(int32_t) * pt.count, hs));
        }
        off += pt.count;
    }
    if (n > 0) {
        kb::k_scatter_out<<<(int)std::min<int64_t>((n + 255) / 256, 16 * kb::sm_count()), 256, 0,
                            hs>>>(n, m->pot_all, m->idx_all, out);
        KB_CHECK_LAUNCH();
    }
}

// Kernels of one execute: the parts' pipelines, two routing passes per part,
// the peer core sums and the final scatter.
int multi_launches(const MultiPlan* m, int64_t n) {
    int l = 0;
    for (auto& pt : m->parts) l += pt.plan->launches + (n > 0 ? 2 : 0);
    if (m->coll == KPME_GPU_COLL_PEER) l += m->G;
    return l + (n > 0 ? 1 : 0);
}

// Sort / cell flags of every part (after its stream drained).
void check_parts(MultiPlan* m) {
    for (auto& pt : m->parts) {
        const kb::DeviceGuard dg(pt.device);
        KB_CUDA(cudaMemcpyAsync(pt.plan->flags_h, pt.plan->sb.bad, 2 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, pt.plan->stream));
        KB_CUDA(cudaStreamSynchronize(pt.plan->stream));
        check_flags(pt.plan->flags_h);
    }
}

}  // namespace

void create_multi(const kpme_gpu_config* cfg, int64_t max_particles, const int dims[3],
                  kpme_gpu_plan* out) {
    validate(cfg);
    if (!out) invalid("kpme_gpu_plan_create: null output");
    const int G = cfg->ndevices;
    if (G < 1 || !cfg->devices) invalid("kpme_gpu: empty device list");
    if (G > kb::PerDevice::kMax) invalid("kpme_gpu: more than 64 device entries");
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1) invalid("kpme_gpu_plan_create_multi: rank grid dims must be >= 1");
    if ((int64_t)dims[0] * dims[1] * dims[2] != G)
        invalid("kpme_gpu_plan_create_multi: rank grid size differs from the device count");
    if (max_particles < 0 || max_particles > INT32_MAX)
        invalid("kpme_gpu_plan_create: particle capacity out of range");
    int ndev = 0;
    KB_CUDA(cudaGetDeviceCount(&ndev));
    for (int d = 0; d < G; ++d)
        if (cfg->devices[d] < 0 || cfg->devices[d] >= ndev)
            invalid("kpme_gpu: device ordinal out of range");
    auto p = new kpme_gpu_plan_s();
    auto m = new MultiPlan();
    p->multi = m;
    try {
        std::copy(dims, dims + 3, m->dims);
        m->G = G;
        m->cap = max_particles;
        p->cap = max_particles;
        p->device = cfg->devices[0];
        m->parts.resize(G);
        // RankGrid::unflatten (parallel.hpp:63-70): rank r -> (r0, r1, r2)
        for (int r = 0; r < G; ++r) {
            const int r2 = r % dims[2], r1 = (r / dims[2]) % dims[1], r0 = r / (dims[2] * dims[1]);
            const int rc[3] = {r0, r1, r2};
            int lo[3], hi[3];
            for (int a = 0; a < 3; ++a) {
                lo[a] = split_lo(cfg->counts[a], rc[a], dims[a]);
                hi[a] = split_lo(cfg->counts[a], rc[a] + 1, dims[a]);
            }
            kpme_gpu_config c = *cfg;
            c.device = cfg->devices[r];
            c.ndevices = 0;
            c.devices = nullptr;
            c.formulation = KPME_GPU_FORM_COLLAPSED;
            Part& pt = m->parts[r];
            pt.device = c.device;
            create_plan(&c, max_particles, lo, hi, &pt.plan);
        }
        const kpme_gpu_plan p0 = m->parts[0].plan;
        p->g = p0->g;
        p->g.x_lo = p->g.y_lo = p->g.z_lo = 0;
        p->g.x_hi = cfg->counts[0];
        p->g.y_hi = cfg->counts[1];
        p->g.z_hi = cfg->counts[2];
        p->nterms = cfg->nterms;
        p->correction = cfg->correction;
        const int R = p0->g.R;
        m->E = R * R * R + 1;
        // peer reachability; enable every distinct pair
        m->peer_ok = true;
        m->distinct = true;
        for (int i = 0; i < G; ++i)
            for (int j = 0; j < G; ++j) {
                const int di = m->parts[i].device, dj = m->parts[j].device;
                if (i != j && di == dj) m->distinct = false;
                if (di == dj) continue;
                int ok = 0;
                KB_CUDA(cudaDeviceCanAccessPeer(&ok, di, dj));
                if (!ok) {
                    m->peer_ok = false;
                    continue;
                }
                const kb::DeviceGuard dg(di);
                const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
                else if (e != cudaSuccess)
                    KB_CUDA(e);
            }
        const int ntiles = (int)std::max<int64_t>(1, (max_particles + kb::kRouteTile - 1) /
                                                         kb::kRouteTile);
        for (auto& pt : m->parts) {
            const kb::DeviceGuard dg(pt.device);
            pt.xyz = pt.alloc<double>((size_t)max_particles * 3);
            pt.q = pt.alloc<double>(max_particles);
            pt.xyz_c = pt.alloc<double>((size_t)max_particles * 3);
            pt.q_c = pt.alloc<double>(max_particles);
            pt.idx = pt.alloc<int32_t>(max_particles);
            pt.tiles = pt.alloc<int32_t>(ntiles);
            pt.count_d = pt.alloc<int64_t>(1);
            pt.bad = pt.alloc<unsigned long long>(1);
            pt.core = pt.alloc<double>(m->E);
            pt.core_sum = pt.alloc<double>(m->E);
            pt.core_ptrs = pt.alloc<const double*>(G);
            pt.pot = pt.alloc<double>(max_particles);
            KB_CUDA(cudaEventCreateWithFlags(&pt.ev_route, cudaEventDisableTiming));
            KB_CUDA(cudaEventCreateWithFlags(&pt.ev_fwd, cudaEventDisableTiming));
            KB_CUDA(cudaEventCreateWithFlags(&pt.ev_bwd, cudaEventDisableTiming));
        }
        std::vector<const double*> cores;
        for (auto& pt : m->parts) cores.push_back(pt.core);
        for (auto& pt : m->parts) {
            const kb::DeviceGuard dg(pt.device);
            KB_CUDA(cudaMemcpy(pt.core_ptrs, cores.data(), sizeof(double*) * G,
                               cudaMemcpyHostToDevice));
        }
        {
            const kb::DeviceGuard dg(m->parts[0].device);
            auto halloc = [&](size_t bytes) {
                void* q = nullptr;
                KB_CUDA(cudaMalloc(&q, std::max<size_t>(bytes, 8)));
                m->home_allocs.push_back(q);
                return q;
            };
            m->pot_all = static_cast<double*>(halloc(sizeof(double) * max_particles));
            m->idx_all = static_cast<int32_t*>(halloc(sizeof(int32_t) * max_particles));
            m->out_home = static_cast<double*>(halloc(sizeof(double) * max_particles));
            KB_CUDA(cudaMallocHost(&m->counts_h, sizeof(int64_t) * G));
            KB_CUDA(cudaMallocHost(&m->bad_h, sizeof(unsigned long long) * G));
        }
        m->coll = m->peer_ok ? KPME_GPU_COLL_PEER : KPME_GPU_COLL_NCCL;
        p->stream = m->parts[0].plan->stream;  // owned by the home part
        p->own_stream = false;
        if (!m->peer_ok && !m->distinct)
            invalid("kpme_gpu: devices without peer access must be distinct (NCCL exchange)");
        *out = p;
    } catch (...) {
        delete p;
        throw;
    }
}

void multi_set_collective(kpme_gpu_plan p, int mode) {
    MultiPlan* m = p->multi;
    if (mode == KPME_GPU_COLL_AUTO) mode = m->peer_ok ? KPME_GPU_COLL_PEER : KPME_GPU_COLL_NCCL;
    if (mode == KPME_GPU_COLL_PEER && !m->peer_ok)
        invalid("kpme_gpu_plan_set_collective: devices lack peer access");
    if (mode == KPME_GPU_COLL_NCCL) {
        if (!m->distinct) invalid("kpme_gpu: the NCCL exchange needs distinct devices");
        init_nccl(m);
    } else if (mode != KPME_GPU_COLL_PEER) {
        invalid("kpme_gpu_plan_set_collective: unknown mode");
    }
    m->coll = mode;
}

int multi_collective(kpme_gpu_plan p) { return p->multi->coll; }

void multi_execute_host(kpme_gpu_plan p, int64_t n, const double* xyz, const double* q,
                        double* out) {
    MultiPlan* m = p->multi;
    if (n > m->cap) invalid("kpme_gpu: more particles than the plan was created for");
    std::vector<const double*> xs(m->G), qs(m->G);
    // every device gets the whole particle set over its own host link
    for (int d = 0; d < m->G; ++d) {
        Part& pt = m->parts[d];
        const kb::DeviceGuard dg(pt.device);
        if (n > 0) {
            KB_CUDA(cudaMemcpyAsync(pt.xyz, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice,
                                    pt.plan->stream));
            KB_CUDA(cudaMemcpyAsync(pt.q, q, sizeof(double) * n, cudaMemcpyHostToDevice,
                                    pt.plan->stream));
        }
        xs[d] = pt.xyz;
        qs[d] = pt.q;
    }
    route_all(m, n, xs.data(), qs.data());
    compute_and_merge(m, n, m->out_home);
    p->launches = multi_launches(m, n);
    Part& home = m->parts[0];
    {
        const kb::DeviceGuard dg(home.device);
        if (n > 0)
            KB_CUDA(cudaMemcpyAsync(out, m->out_home, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                    home.plan->stream));
    }
    check_parts(m);
}

void multi_execute_device(kpme_gpu_plan p, int64_t n, const double* xyz, const double* q,
                          double* out, int flags) {
    MultiPlan* m = p->multi;
    if (n > m->cap) invalid("kpme_gpu: more particles than the plan was created for");
    std::vector<const double*> xs(m->G), qs(m->G);
    Part& home = m->parts[0];
    {
        // the caller's buffers live on the home device; order after its work
        const kb::DeviceGuard dg(home.device);
        KB_CUDA(cudaEventRecord(home.ev_bwd, home.plan->stream));
    }
    for (int d = 0; d < m->G; ++d) {
        Part& pt = m->parts[d];
        const kb::DeviceGuard dg(pt.device);
        if (pt.device == home.device) {
            xs[d] = xyz;
            qs[d] = q;
            if (d) KB_CUDA(cudaStreamWaitEvent(pt.plan->stream, home.ev_bwd, 0));
            continue;
        }
        KB_CUDA(cudaStreamWaitEvent(pt.plan->stream, home.ev_bwd, 0));
        if (n > 0) {
            KB_CUDA(cudaMemcpyPeerAsync(pt.xyz, pt.device, xyz, home.device,
                                        sizeof(double) * 3 * n, pt.plan->stream));
            KB_CUDA(cudaMemcpyPeerAsync(pt.q, pt.device, q, home.device, sizeof(double) * n,
                                        pt.plan->stream));
        }
        xs[d] = pt.xyz;
        qs[d] = pt.q;
    }
    route_all(m, n, xs.data(), qs.data());
    compute_and_merge(m, n, out);
    p->launches = multi_launches(m, n);
    if (!(flags & KPME_GPU_DEFER_CHECKS)) check_parts(m);
}

void multi_status(kpme_gpu_plan p) { check_parts(p->multi); }

std::vector<int> multi_devices(kpme_gpu_plan p) {
    if (!p->multi) return {p->device};
    std::vector<int> d;
    for (auto& pt : p->multi->parts) d.push_back(pt.device);
    return d;
}

void multi_set_home_stream(kpme_gpu_plan p, cudaStream_t s) {
    kpme_gpu_plan home = p->multi->parts[0].plan;
    const int st = kpme_gpu_plan_set_stream(home, s);
    if (st) throw kb::Error(st, kb::g_last_error);
    p->stream = home->stream;
}

}  // namespace kbp
