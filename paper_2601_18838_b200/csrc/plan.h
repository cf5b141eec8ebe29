// plan.h -- the plan object behind kpme_gpu_plan and the helpers shared by
// plan.cu (single-device pipeline) and multi.cu (multi-device plans).
// Not part of the ABI.
#pragma once

#include <nccl.h>

#include <string>
#include <vector>

#include "internal.h"

namespace kb {
extern thread_local std::string g_last_error;
struct MultiPlan;
void destroy_multi(MultiPlan* m);
}  // namespace kb

// Particle chunks of the pipelined host path (kpme_gpu_plan_execute).
constexpr int kMaxChunks = 8;

struct kpme_gpu_plan_s {
    kb::Geometry g{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t cap = 0;
    int nterms = 0;
    double correction = 0.0;
    int S = 1;
    int form = KPME_GPU_FORM_COLLAPSED;
    int launches = 0;
    int64_t last_n = 0;
    const double* last_xyz = nullptr;  // inputs of the last forward half (direct records)
    const double* last_q = nullptr;
    bool use_sort2 = false;
    // hot path reads particle records through perm from the inputs (no sorted
    // copy written by the sort; ColumnArgs::direct)
    bool direct = false;

    // factor tables
    double* tw = nullptr;
    double* prof = nullptr;
    double* W[3] = {nullptr, nullptr, nullptr};
    double* WL[3] = {nullptr, nullptr, nullptr};  // W_a Lambda (monomial hot path)
    double* lam = nullptr;
    double4* cellax = nullptr;  // [K0 + K1 + K2] (lo, hi, mid, 1/half)
    double* D = nullptr;
    double* G = nullptr;
    // collapsed-core work
    double* T1 = nullptr;
    double* T2 = nullptr;
    double* F = nullptr;
    double* B2 = nullptr;
    double* colq = nullptr;
    double* corr = nullptr;
    double* Fpart = nullptr;
    // sort
    kb::SortBuffers sb{};
    double4* sp = nullptr;
    // host-buffer staging
    double* xyz_d = nullptr;
    double* q_d = nullptr;
    double* out_d = nullptr;
    unsigned long long* flags_h = nullptr;  // pinned
    // chunked host path (kpme_gpu_plan_execute): copies on their own stream,
    // one independent sort + spread per particle chunk
    int host_chunks = -1;                   // -1: automatic
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_out[kMaxChunks] = {};
    int32_t* cstart = nullptr;              // [kMaxChunks][ncell + 1]
    unsigned long long* cbad = nullptr;     // [kMaxChunks][2]
    unsigned long long* cflags_h = nullptr; // pinned [kMaxChunks][2]
    double* cFpart = nullptr;               // [R^3 + 1][kMaxChunks * S * ncol]
    // dense form
    double* A[3] = {nullptr, nullptr, nullptr};
    double* cells = nullptr;
    double* mesh_in = nullptr;
    double* mesh_out = nullptr;
    double* work = nullptr;
    size_t work_bytes = 0;
    // multi-process decomposition: this rank's NCCL communicator (owned);
    // execute sums the partial cores over it between the two halves
    ncclComm_t comm = nullptr;
    int comm_ranks = 1;
    // multi-device plan (one process, several devices; multi.cu): the plan
    // is a group of block plans and every call dispatches to it
    kb::MultiPlan* multi = nullptr;
    // graph
    cudaGraphExec_t gexec = nullptr;
    int64_t g_n = -1;
    const void* g_ptr[3] = {nullptr, nullptr, nullptr};
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    std::vector<double> stage_ms;
    std::vector<void*> allocs;

    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        KB_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    ~kpme_gpu_plan_s() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (gexec) cudaGraphExecDestroy(gexec);
        for (int c = 0; c < kMaxChunks; ++c) {
            if (ev_in[c]) cudaEventDestroy(ev_in[c]);
            if (ev_out[c]) cudaEventDestroy(ev_out[c]);
        }
        if (cstream) cudaStreamDestroy(cstream);
        if (cflags_h) cudaFreeHost(cflags_h);
        for (auto e : ev) cudaEventDestroy(e);
        for (void* p : allocs) cudaFree(p);
        if (flags_h) cudaFreeHost(flags_h);
        if (comm) ncclCommDestroy(comm);
        if (own_stream && stream) cudaStreamDestroy(stream);
        if (prev >= 0) cudaSetDevice(prev);
        if (multi) kb::destroy_multi(multi);
    }
};

namespace kbp {
using kb::Error;


template <class F>
inline int guarded(F&& f) {
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

[[noreturn]] inline void invalid(const char* msg) { throw Error(KPME_GPU_INVALID_ARGUMENT, msg); }

// plan.cu
void need_single(kpme_gpu_plan p);
void validate(const kpme_gpu_config* c);
void create_plan(const kpme_gpu_config* cfg, int64_t max_particles, const int lo[3],
                 const int hi[3], kpme_gpu_plan* out);
void reset_flags(kpme_gpu_plan p);
void check_flags(const unsigned long long* f);
void forward_half(kpme_gpu_plan p, int64_t n, const double* xyz, const double* q, double* core);
void backward_half(kpme_gpu_plan p, const double* core, double* out);
// the balanced contiguous split of k cells over parts (dist.slab_bounds)
inline int split_lo(int k, int i, int parts) { return (int)((int64_t)k * i / parts); }

// multi.cu
void create_multi(const kpme_gpu_config* cfg, int64_t max_particles, const int dims[3],
                  kpme_gpu_plan* out);
void multi_execute_host(kpme_gpu_plan p, int64_t n, const double* xyz, const double* q,
                        double* out);
void multi_execute_device(kpme_gpu_plan p, int64_t n, const double* xyz, const double* q,
                          double* out, int flags);
void multi_status(kpme_gpu_plan p);
std::vector<int> multi_devices(kpme_gpu_plan p);
void multi_set_home_stream(kpme_gpu_plan p, cudaStream_t s);
void multi_set_collective(kpme_gpu_plan p, int mode);
int multi_collective(kpme_gpu_plan p);
}  // namespace kbp
