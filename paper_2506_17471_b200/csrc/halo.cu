// halo.cu — the exchange step of the cell-partitioned multi-GPU action, GPU to GPU.
//
// One process (or thread) per GPU owns a slab of cells and a compact local instance.  Per action:
//   pull      ghost trial-space nodes are read straight from their owners' input buffers
//   boundary  the cells touching shared rows (the local cell order puts them first) compute
//   push      their partial sums of rows owned elsewhere are stored into the owners' receive
//             buffers (side stream: overlaps the interior cells)
//   interior  the remaining cells compute
//   complete  each owned shared row adds what it received, in ascending rank order (deterministic)
// Peer buffers are reached over NVLink with plain loads/stores: opened with CUDA IPC across
// processes, used directly within one process (peer access across devices).  Ranks are ordered by
// device-side flags (release/acquire at system scope) instead of host synchronisation, so a step
// is a fixed sequence of launches on one stream with no host round trip.  Every wait is bounded
// (FEMGPU_HALO_TIMEOUT_MS, default 20 s on %globaltimer): a missing peer sets an error flag that
// femgpu_halo_check reports, and the GPU never hangs.
//
// Flags of rank r (int64, in r's memory; peers write the `pushed` slots):
//   [0] xready   the step whose owned inputs r has published (written by r)
//   [1] consumed the step whose received contributions r has added (written by r)
//   [2..5] error: which wait timed out (1 pull, 2 push, 4 receive), the peer, value seen, wanted
//   [6] step     this rank's step counter, advanced on the device by the first kernel of a step (so a
//                captured CUDA graph of one step replays correctly)
//   [8 + q]      pushed: the step whose contributions rank q has stored into r's receive buffer
// Receive buffers are double-buffered by step parity; a push of step k waits until the owner
// consumed step k - 2, so a fast rank cannot overwrite contributions still being added.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>
#include <unistd.h>

#include "femgpu_internal.hpp"

namespace {

constexpr int kMaxWorld = 64;
constexpr int kFlagPushed = 8;
constexpr int kFlagStep = 6;
constexpr int kRed = kFlagPushed + kMaxWorld;     // all-reduce slots: [parity][source rank][value bits, epoch]
constexpr int kFlagWords = kRed + 4 * kMaxWorld;
constexpr int kMaxSpaces = 2 * FEMGPU_MAX_SPACES;

__device__ __forceinline__ long long ld_acquire(const long long* p) {
    long long v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(long long* p, long long v) {
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spins (one thread) until *p >= want or the timeout; on timeout records in the local error
// words which wait (bit `what`: 1 pull, 2 push, 4 receive), on which peer, and the value seen.
__device__ void wait_geq(const long long* p, long long want, long long* err, unsigned long long timeout_ns, int what,
                         int peer) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    long long v;
    while ((v = ld_acquire(p)) < want) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
            atomicOr(reinterpret_cast<unsigned long long*>(err), static_cast<unsigned long long>(what));
            err[1] = peer;
            err[2] = v;
            err[3] = want;
            return;
        }
        __nanosleep(200);
    }
}

struct PullArgs {
    long long* my_flags;
    const long long* const* peer_flags;  // [world] (device table)
    const int* pull_peers;               // distinct peers to wait for
    int n_pull_peers;
    long long step;
    unsigned long long timeout_ns;
    // entries
    long long n;
    const int* space;
    const int* peer;
    const int* node;
    const int* remote;
    double* const* my_x;                 // [kMaxSpaces]
    const double* const* peer_x;         // [world * kMaxSpaces]
    const int* stride;                   // [kMaxSpaces] doubles per node in the device layout
    const int* comps;                    // [kMaxSpaces] components per node
};

__device__ __forceinline__ long long cur_step(const long long* flags) {
    return *reinterpret_cast<const volatile long long*>(flags + kFlagStep);
}

__global__ void bump_step_kernel(long long* flags) { flags[kFlagStep] += 1; }

__global__ void pull_kernel(PullArgs a) {
    a.step = cur_step(a.my_flags);
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            __threadfence_system();  // the caller's updates of the owned inputs precede the flag
            st_release(a.my_flags + 0, a.step);
        }
        for (int i = 0; i < a.n_pull_peers; ++i)
            wait_geq(a.peer_flags[a.pull_peers[i]] + 0, a.step, a.my_flags + 2, a.timeout_ns, 1, a.pull_peers[i]);
    }
    __syncthreads();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < a.n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int s = a.space[i], st = a.stride[s];
        const double* src = a.peer_x[a.peer[i] * kMaxSpaces + s] + static_cast<long long>(a.remote[i]) * st;
        double* dst = a.my_x[s] + static_cast<long long>(a.node[i]) * st;
        for (int c = 0; c < a.comps[s]; ++c) dst[c] = src[c];
    }
}

struct PushArgs {
    long long* my_flags;
    long long* const* peer_flags;  // [world]
    const int* targets;            // distinct owners pushed to
    int n_targets;
    int rank;
    long long step;
    unsigned long long timeout_ns;
    long long n;
    const int* row;                // local rows
    const long long* dst_off;      // element offset in the owner's receive buffer (parity 0)
    const int* dst_peer;
    double* const* peer_recv;      // [world] receive buffer base of each owner
    const long long* peer_slot;    // [world] parity stride (receive-buffer length) of each owner
    const double* y;
    unsigned int* done;            // block counter (local)
};

__global__ void push_kernel(PushArgs a) {
    a.step = cur_step(a.my_flags);
    if (threadIdx.x == 0)  // slot reuse: the owner must have consumed step - 2
        for (int i = 0; i < a.n_targets; ++i)
            wait_geq(a.peer_flags[a.targets[i]] + 1, a.step - 2, a.my_flags + 2, a.timeout_ns, 2, a.targets[i]);
    __syncthreads();
    const long long par = a.step & 1;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < a.n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int q = a.dst_peer[i];
        a.peer_recv[q][par * a.peer_slot[q] + a.dst_off[i]] = a.y[a.row[i]];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(a.done, 1u);
        if (prev == gridDim.x - 1) {  // last block: every contribution of this step is stored
            *a.done = 0;
            __threadfence_system();
            for (int i = 0; i < a.n_targets; ++i) st_release(a.peer_flags[a.targets[i]] + kFlagPushed + a.rank, a.step);
        }
    }
}

struct RecvArgs {
    long long* my_flags;
    const int* sources;      // distinct ranks that push to me
    int n_sources;
    long long step;
    unsigned long long timeout_ns;
    long long n_rows;
    const int* row;          // owned rows receiving contributions
    const long long* ptr;    // CSR over the receive buffer: row i adds recv[pos[ptr[i]..ptr[i+1])]
    const long long* pos;    //   positions in ascending source rank
    const double* recv;      // my receive buffer
    long long slot;          // parity stride
    double* y;
    unsigned int* done;
};

__global__ void recv_kernel(RecvArgs a) {
    a.step = cur_step(a.my_flags);
    if (threadIdx.x == 0)
        for (int i = 0; i < a.n_sources; ++i)
            wait_geq(a.my_flags + kFlagPushed + a.sources[i], a.step, a.my_flags + 2, a.timeout_ns, 4, a.sources[i]);
    __syncthreads();
    const double* r = a.recv + (a.step & 1) * a.slot;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < a.n_rows;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double acc = a.y[a.row[i]];
        for (long long k = a.ptr[i]; k < a.ptr[i + 1]; ++k) acc += r[a.pos[k]];
        a.y[a.row[i]] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(a.done, 1u);
        if (prev == gridDim.x - 1) {
            *a.done = 0;
            __threadfence_system();
            st_release(a.my_flags + 1, a.step);
        }
    }
}

// ---- device-side all-reduce (sum of one double over the ranks) through the peers' flag words: rank r
// stores its value into slot r of every rank's flags (double-buffered by the epoch's parity), then a
// release of the epoch; each rank acquires every slot's epoch and sums the values in rank order
// (deterministic).  One thread; bounded waits like the exchange (error bit 8).
__global__ void allreduce_kernel(long long* const* peer_flags, long long* my_flags, int rank, int world,
                                 const double* in, double* out, long long epoch, unsigned long long timeout_ns) {
    const int par = static_cast<int>(epoch & 1);
    const long long bits = __double_as_longlong(*in);
    for (int q = 0; q < world; ++q) {
        long long* slot = peer_flags[q] + kRed + par * 2 * kMaxWorld + 2 * rank;
        slot[0] = bits;
        st_release(slot + 1, epoch);
    }
    double sum = 0.0;
    for (int q = 0; q < world; ++q) {
        const long long* slot = my_flags + kRed + par * 2 * kMaxWorld + 2 * q;
        wait_geq(slot + 1, epoch, my_flags + 2, timeout_ns, 8, q);
        sum += __longlong_as_double(*(volatile const long long*)slot);
    }
    *out = sum;
}

constexpr int kCgBlocks = 1184, kCgThreads = 256;

__device__ __forceinline__ void cg_block_sum(double v, double* out) {
    __shared__ double red[kCgThreads];
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = kCgThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

#define CG_LOOP(i, n) for (long long i = blockIdx.x * (long long)kCgThreads + threadIdx.x; i < (n); i += (long long)kCgBlocks * kCgThreads)

__global__ void cg_mask_dot(const double* a, const double* b, const unsigned char* owned, long long n, double* part) {
    double s = 0.0;
    CG_LOOP(i, n) if (owned[i]) s += a[i] * b[i];
    cg_block_sum(s, part + blockIdx.x);
}
__global__ void cg_final(const double* part, double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < kCgBlocks; i += kCgThreads) s += part[i];
    cg_block_sum(s, out);
}
// r = owned ? b - ax : 0; p = r
__global__ void cg_init(double* r, double* p, const double* b, const double* ax, const unsigned char* owned, long long n) {
    CG_LOOP(i, n) {
        const double ri = owned[i] ? b[i] - ax[i] : 0.0;
        r[i] = ri;
        p[i] = ri;
    }
}
// ghost rows of A p hold partial sums: zero them (only owned rows are the product)
__global__ void cg_mask(double* v, const unsigned char* owned, long long n) {
    CG_LOOP(i, n) if (!owned[i]) v[i] = 0.0;
}
__global__ void cg_update_xr(double* x, double* r, const double* p, const double* ap, const unsigned char* owned, long long n,
                             const double* rr, const double* pap, double* part) {
    const double alpha = *rr / *pap;
    double s = 0.0;
    CG_LOOP(i, n) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        if (owned[i]) s += ri * ri;
    }
    cg_block_sum(s, part + blockIdx.x);
}
__global__ void cg_update_p(double* p, const double* r, long long n, const double* rr_new, const double* rr_old) {
    const double beta = *rr_new / *rr_old;
    CG_LOOP(i, n) p[i] = r[i] + beta * p[i];
}

// What one rank publishes: IPC handles of its flags, receive buffer and input buffers, plus raw
// pointers for peers in the same process.
struct Export {
    int32_t magic = 0x68616c6f, rank = 0, device = 0, pid = 0;
    int32_t n_x = 0, pad_ = 0;
    long long recv_total = 0;
    long long recv_off[kMaxWorld] = {};  // offset of each source's segment in my receive buffer
    cudaIpcMemHandle_t h_flags{}, h_recv{}, h_x[kMaxSpaces]{};
    unsigned long long raw_flags = 0, raw_recv = 0, raw_x[kMaxSpaces] = {};
};

template <typename T>
T* dev_copy(const std::vector<T>& v, std::vector<void*>& keep) {
    if (v.empty()) return nullptr;
    void* p = nullptr;
    FG_CUDA(cudaMalloc(&p, v.size() * sizeof(T)));
    FG_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    keep.push_back(p);
    return static_cast<T*>(p);
}

}  // namespace

struct femgpu_halo {
    femgpu::Instance* inst = nullptr;
    int rank = 0, world = 1, boundary = 0, device = 0;
    long long step = 0;
    unsigned long long timeout_ns = 20000000000ULL;
    std::vector<void*> keep;           // device allocations owned here
    long long* flags = nullptr;
    double* recv = nullptr;
    long long recv_total = 0;
    std::vector<long long> recv_off;   // per source rank
    unsigned int* counters = nullptr;  // [0] push blocks, [1] recv blocks
    cudaStream_t side = nullptr;
    cudaEvent_t ev_boundary = nullptr, ev_pushed = nullptr;
    // host-side plan
    std::vector<int> push_row, push_peer, pull_space, pull_peer, pull_node, pull_remote, recv_sources, push_targets,
        pull_peers;
    std::vector<long long> push_local_idx;  // position of each push entry inside its (rank -> owner) segment
    std::vector<int> recv_row_u;
    std::vector<long long> recv_ptr, recv_pos;
    // device-side plan
    int *d_push_row = nullptr, *d_push_peer = nullptr, *d_targets = nullptr, *d_pull_space = nullptr,
        *d_pull_peer = nullptr, *d_pull_node = nullptr, *d_pull_remote = nullptr, *d_pull_peers = nullptr,
        *d_recv_row = nullptr, *d_sources = nullptr, *d_stride = nullptr, *d_comps = nullptr;
    long long *d_push_off = nullptr, *d_recv_ptr = nullptr, *d_recv_pos = nullptr, *d_peer_slot = nullptr;
    long long** d_peer_flags = nullptr;
    double** d_peer_recv = nullptr;
    double** d_my_x = nullptr;
    const double** d_peer_x = nullptr;
    std::vector<void*> opened;  // IPC-opened peer allocations
    bool imported = false;
    long long red_epoch = 0;    // device all-reduces issued (identical sequence on every rank)
    unsigned char* d_owned = nullptr;  // rows this rank owns (not pushed elsewhere)
    std::vector<double*> cg_work;      // r, p, ap, partials + scalars

    ~femgpu_halo() {
        cudaSetDevice(device);
        if (side) cudaStreamSynchronize(side);
        if (inst) cudaStreamSynchronize(inst->stream);
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        for (void* p : keep) cudaFree(p);
        if (side) cudaStreamDestroy(side);
        if (ev_boundary) cudaEventDestroy(ev_boundary);
        if (ev_pushed) cudaEventDestroy(ev_pushed);
    }
};

namespace {

void halo_step(femgpu_halo& H, const femgpu::KernelPlan& kp, double* y, cudaStream_t s) {
    femgpu::Instance& I = *H.inst;
    ++H.step;  // host mirror (messages); the kernels read the device counter
    bump_step_kernel<<<1, 1, 0, s>>>(H.flags);
    FG_CUDA(cudaGetLastError());
    FG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * static_cast<size_t>(I.output_size), s));
    {  // publish my inputs, pull the ghosts (always launched: peers wait for my xready)
        PullArgs a{};
        a.my_flags = H.flags;
        a.peer_flags = const_cast<const long long* const*>(H.d_peer_flags);
        a.pull_peers = H.d_pull_peers;
        a.n_pull_peers = static_cast<int>(H.pull_peers.size());
        a.timeout_ns = H.timeout_ns;
        a.n = static_cast<long long>(H.pull_node.size());
        a.space = H.d_pull_space;
        a.peer = H.d_pull_peer;
        a.node = H.d_pull_node;
        a.remote = H.d_pull_remote;
        a.my_x = H.d_my_x;
        a.peer_x = H.d_peer_x;
        a.stride = H.d_stride;
        a.comps = H.d_comps;
        const int blocks = static_cast<int>(std::max(1LL, std::min(148LL, (a.n + 255) / 256)));
        pull_kernel<<<blocks, 256, 0, s>>>(a);
        FG_CUDA(cudaGetLastError());
    }
    const bool split = H.boundary > 0 && H.boundary < I.cells && femgpu::supports_cell_range(kp);
    if (split) femgpu::run_action_range(I, kp, y, s, 0, H.boundary, false);
    else femgpu::run_action_range(I, kp, y, s, 0, I.cells, false);
    // push the partial sums of rows owned elsewhere (side stream: overlaps the interior cells)
    if (!H.push_targets.empty()) {
        FG_CUDA(cudaEventRecord(H.ev_boundary, s));
        FG_CUDA(cudaStreamWaitEvent(H.side, H.ev_boundary, 0));
        PushArgs a{};
        a.my_flags = H.flags;
        a.peer_flags = H.d_peer_flags;
        a.targets = H.d_targets;
        a.n_targets = static_cast<int>(H.push_targets.size());
        a.rank = H.rank;
        a.timeout_ns = H.timeout_ns;
        a.n = static_cast<long long>(H.push_row.size());
        a.row = H.d_push_row;
        a.dst_off = H.d_push_off;
        a.dst_peer = H.d_push_peer;
        a.peer_recv = H.d_peer_recv;
        a.peer_slot = H.d_peer_slot;
        a.y = y;
        a.done = H.counters;
        const int blocks = static_cast<int>(std::max(1LL, std::min(148LL, (a.n + 255) / 256)));
        push_kernel<<<blocks, 256, 0, H.side>>>(a);
        FG_CUDA(cudaGetLastError());
        FG_CUDA(cudaEventRecord(H.ev_pushed, H.side));
    }
    if (split) femgpu::run_action_range(I, kp, y, s, H.boundary, I.cells, false);
    {  // complete the owned shared rows (always launched: pushers wait for my consumed flag)
        RecvArgs a{};
        a.my_flags = H.flags;
        a.sources = H.d_sources;
        a.n_sources = static_cast<int>(H.recv_sources.size());
        a.timeout_ns = H.timeout_ns;
        a.n_rows = static_cast<long long>(H.recv_row_u.size());
        a.row = H.d_recv_row;
        a.ptr = H.d_recv_ptr;
        a.pos = H.d_recv_pos;
        a.recv = H.recv;
        a.slot = H.recv_total;
        a.y = y;
        a.done = H.counters + 1;
        const int blocks = static_cast<int>(std::max(1LL, std::min(148LL, (a.n_rows + 255) / 256)));
        recv_kernel<<<blocks, 256, 0, s>>>(a);
        FG_CUDA(cudaGetLastError());
    }
    if (!H.push_targets.empty()) FG_CUDA(cudaStreamWaitEvent(s, H.ev_pushed, 0));
    // bump + pull + action launch(es) + push + completion (the memset is the driver's)
    I.last_launches = 3 + (split ? 2 : 1) + (H.push_targets.empty() ? 0 : 1);
}

}  // namespace

extern "C" {

femgpu_status femgpu_halo_create(femgpu_instance* inst, int32_t rank, int32_t world, int32_t boundary_cells,
                                 int64_t n_push, const int32_t* push_peer, const int32_t* push_row, int64_t n_recv,
                                 const int32_t* recv_peer, const int32_t* recv_row, int64_t n_pull,
                                 const int32_t* pull_space, const int32_t* pull_peer, const int32_t* pull_node,
                                 const int32_t* pull_remote, femgpu_halo** out) {
    return femgpu::abi_guard([&] {
        if (!inst || !inst->impl || !out) femgpu::invalid("halo: null argument");
        if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world) femgpu::invalid("halo: rank/world out of range");
        femgpu::Instance& I = *inst->impl;
        if (boundary_cells < 0 || boundary_cells > I.cells) femgpu::invalid("halo: boundary cell count out of range");
        auto H = std::make_unique<femgpu_halo>();
        H->inst = &I;
        H->rank = rank;
        H->world = world;
        H->boundary = boundary_cells;
        H->device = I.device;
        if (const char* e = std::getenv("FEMGPU_HALO_TIMEOUT_MS")) H->timeout_ns = std::strtoull(e, nullptr, 10) * 1000000ULL;
        FG_CUDA(cudaSetDevice(I.device));
        const int ns = static_cast<int>(I.sspaces.size()), nv = static_cast<int>(I.vspaces.size());
        auto in_range = [](int v, int hi) { return v >= 0 && v < hi; };
        // push entries grouped by owner (stable: the caller's order inside each owner's segment)
        std::vector<long long> order(static_cast<size_t>(n_push));
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](long long a, long long b) { return push_peer[a] < push_peer[b]; });
        std::vector<long long> seg(world, 0);
        for (long long i : order) {
            const int q = push_peer[i];
            if (!in_range(q, world) || q == rank || !in_range(push_row[i], I.output_size))
                femgpu::invalid("halo: push entry out of range");
            H->push_peer.push_back(q);
            H->push_row.push_back(push_row[i]);
            H->push_local_idx.push_back(seg[q]++);
        }
        for (int q = 0; q < world; ++q)
            if (seg[q]) H->push_targets.push_back(q);
        // receive buffer: one segment per source rank (ascending), entries in the source's push order
        H->recv_off.assign(world, 0);
        std::vector<long long> cnt(world, 0);
        for (long long i = 0; i < n_recv; ++i) {
            if (!in_range(recv_peer[i], world) || recv_peer[i] == rank || !in_range(recv_row[i], I.output_size))
                femgpu::invalid("halo: receive entry out of range");
            ++cnt[recv_peer[i]];
        }
        long long off = 0;
        for (int q = 0; q < world; ++q) {
            H->recv_off[q] = off;
            off += cnt[q];
            if (cnt[q]) H->recv_sources.push_back(q);
        }
        H->recv_total = std::max(1LL, off);
        // CSR per receiving row, sources ascending (fixed summation order)
        std::vector<long long> fill(H->recv_off.begin(), H->recv_off.end());
        std::vector<std::pair<int, long long>> rp;  // (row, position), stable in source order
        std::vector<long long> ord(static_cast<size_t>(n_recv));
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](long long a, long long b) { return recv_peer[a] < recv_peer[b]; });
        for (long long i : ord) rp.push_back({recv_row[i], fill[recv_peer[i]]++});
        std::stable_sort(rp.begin(), rp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t i = 0; i < rp.size(); ++i) {
            if (i == 0 || rp[i].first != rp[i - 1].first) {
                H->recv_row_u.push_back(rp[i].first);
                H->recv_ptr.push_back(static_cast<long long>(i));
            }
            H->recv_pos.push_back(rp[i].second);
        }
        H->recv_ptr.push_back(static_cast<long long>(rp.size()));
        // pulls
        std::vector<char> pull_from(world, 0);
        for (long long i = 0; i < n_pull; ++i) {
            const int s = pull_space[i];
            if (!in_range(s, ns + nv) || !in_range(pull_peer[i], world) || pull_peer[i] == rank)
                femgpu::invalid("halo: pull entry out of range");
            const int glob = s < ns ? I.sspaces[s].global : I.vspaces[s - ns].global;
            if (!in_range(pull_node[i], glob) || pull_remote[i] < 0) femgpu::invalid("halo: pull node out of range");
            H->pull_space.push_back(s);
            H->pull_peer.push_back(pull_peer[i]);
            H->pull_node.push_back(pull_node[i]);
            H->pull_remote.push_back(pull_remote[i]);
            pull_from[pull_peer[i]] = 1;
        }
        for (int q = 0; q < world; ++q)
            if (pull_from[q]) H->pull_peers.push_back(q);
        // device buffers
        {
            void* p = nullptr;
            FG_CUDA(cudaMalloc(&p, kFlagWords * sizeof(long long)));
            FG_CUDA(cudaMemset(p, 0, kFlagWords * sizeof(long long)));
            H->keep.push_back(p);
            H->flags = static_cast<long long*>(p);
            FG_CUDA(cudaMalloc(&p, 2 * static_cast<size_t>(H->recv_total) * sizeof(double)));
            FG_CUDA(cudaMemset(p, 0, 2 * static_cast<size_t>(H->recv_total) * sizeof(double)));
            H->keep.push_back(p);
            H->recv = static_cast<double*>(p);
            FG_CUDA(cudaMalloc(&p, 2 * sizeof(unsigned int)));
            FG_CUDA(cudaMemset(p, 0, 2 * sizeof(unsigned int)));
            H->keep.push_back(p);
            H->counters = static_cast<unsigned int*>(p);
        }
        H->d_push_row = dev_copy(H->push_row, H->keep);
        H->d_push_peer = dev_copy(H->push_peer, H->keep);
        H->d_targets = dev_copy(H->push_targets, H->keep);
        H->d_pull_space = dev_copy(H->pull_space, H->keep);
        H->d_pull_peer = dev_copy(H->pull_peer, H->keep);
        H->d_pull_node = dev_copy(H->pull_node, H->keep);
        H->d_pull_remote = dev_copy(H->pull_remote, H->keep);
        H->d_pull_peers = dev_copy(H->pull_peers, H->keep);
        H->d_recv_row = dev_copy(H->recv_row_u, H->keep);
        H->d_recv_ptr = dev_copy(H->recv_ptr, H->keep);
        H->d_recv_pos = dev_copy(H->recv_pos, H->keep);
        H->d_sources = dev_copy(H->recv_sources, H->keep);
        std::vector<int> stride(kMaxSpaces, 1), comps(kMaxSpaces, 1);
        std::vector<double*> my_x(kMaxSpaces, nullptr);
        for (int s = 0; s < ns; ++s) my_x[s] = I.sspaces[s].d_x;
        for (int s = 0; s < nv; ++s) {
            my_x[ns + s] = I.vspaces[s].d_x;
            stride[ns + s] = femgpu::vec_stride(I.sig.dim);
            comps[ns + s] = I.sig.dim;
        }
        H->d_stride = dev_copy(stride, H->keep);
        H->d_comps = dev_copy(comps, H->keep);
        H->d_my_x = dev_copy(my_x, H->keep);
        // load the exchange kernels now (lazy module loading would otherwise load them at the first
        // launch, which may wait for the device while a peer spins on this rank)
        for (const void* k : {reinterpret_cast<const void*>(pull_kernel), reinterpret_cast<const void*>(push_kernel),
                              reinterpret_cast<const void*>(recv_kernel), reinterpret_cast<const void*>(bump_step_kernel),
                              reinterpret_cast<const void*>(allreduce_kernel), reinterpret_cast<const void*>(cg_mask_dot),
                              reinterpret_cast<const void*>(cg_final), reinterpret_cast<const void*>(cg_init),
                              reinterpret_cast<const void*>(cg_mask), reinterpret_cast<const void*>(cg_update_xr),
                              reinterpret_cast<const void*>(cg_update_p)}) {
            cudaFuncAttributes fa{};
            FG_CUDA(cudaFuncGetAttributes(&fa, k));
        }
        FG_CUDA(cudaStreamCreateWithFlags(&H->side, cudaStreamNonBlocking));
        FG_CUDA(cudaEventCreateWithFlags(&H->ev_boundary, cudaEventDisableTiming));
        FG_CUDA(cudaEventCreateWithFlags(&H->ev_pushed, cudaEventDisableTiming));
        *out = H.release();
    });
}

femgpu_status femgpu_halo_destroy(femgpu_halo* h) {
    return femgpu::abi_guard([&] { delete h; });
}

femgpu_status femgpu_halo_export(femgpu_halo* h, void* buf, size_t cap, size_t* len) {
    return femgpu::abi_guard([&] {
        if (!h) femgpu::invalid("halo: null handle");
        if (len) *len = sizeof(Export);
        if (!buf) return;
        if (cap < sizeof(Export)) femgpu::invalid("halo: export buffer too small");
        FG_CUDA(cudaSetDevice(h->device));
        femgpu::Instance& I = *h->inst;
        Export e;
        e.rank = h->rank;
        e.device = h->device;
        e.pid = static_cast<int32_t>(::getpid());
        e.recv_total = h->recv_total;
        for (int q = 0; q < h->world; ++q) e.recv_off[q] = h->recv_off[q];
        FG_CUDA(cudaIpcGetMemHandle(&e.h_flags, h->flags));
        FG_CUDA(cudaIpcGetMemHandle(&e.h_recv, h->recv));
        e.raw_flags = reinterpret_cast<unsigned long long>(h->flags);
        e.raw_recv = reinterpret_cast<unsigned long long>(h->recv);
        const int ns = static_cast<int>(I.sspaces.size()), nv = static_cast<int>(I.vspaces.size());
        e.n_x = ns + nv;
        for (int s = 0; s < ns + nv; ++s) {
            double* x = s < ns ? I.sspaces[s].d_x : I.vspaces[s - ns].d_x;  // allocation bases (Instance::alloc)
            FG_CUDA(cudaIpcGetMemHandle(&e.h_x[s], x));
            e.raw_x[s] = reinterpret_cast<unsigned long long>(x);
        }
        std::memcpy(buf, &e, sizeof e);
    });
}

femgpu_status femgpu_halo_import(femgpu_halo* h, const void* all, size_t stride) {
    return femgpu::abi_guard([&] {
        if (!h || !all) femgpu::invalid("halo: null argument");
        if (stride < sizeof(Export)) femgpu::invalid("halo: export stride too small");
        if (h->imported) femgpu::invalid("halo: already imported");
        FG_CUDA(cudaSetDevice(h->device));
        const int W = h->world, me = h->rank;
        std::vector<long long*> pflags(W, nullptr);
        std::vector<double*> precv(W, nullptr);
        std::vector<const double*> px(static_cast<size_t>(W) * kMaxSpaces, nullptr);
        std::vector<long long> pslot(W, 1);
        std::vector<long long> push_off(h->push_row.size(), 0);
        const int pid = static_cast<int>(::getpid());
        for (int q = 0; q < W; ++q) {
            Export e;
            std::memcpy(&e, static_cast<const char*>(all) + static_cast<size_t>(q) * stride, sizeof e);
            if (e.magic != 0x68616c6f || e.rank != q) femgpu::invalid("halo: malformed export of rank " + std::to_string(q));
            pslot[q] = e.recv_total;
            if (q == me) {
                pflags[q] = h->flags;
                precv[q] = h->recv;
                continue;
            }
            if (e.pid == pid) {  // same process: the raw pointers are valid here (peer access across devices)
                if (e.device != h->device) {
                    const cudaError_t pe = cudaDeviceEnablePeerAccess(e.device, 0);
                    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) FG_CUDA(pe);
                    cudaGetLastError();
                }
                pflags[q] = reinterpret_cast<long long*>(e.raw_flags);
                precv[q] = reinterpret_cast<double*>(e.raw_recv);
                for (int s = 0; s < e.n_x; ++s) px[static_cast<size_t>(q) * kMaxSpaces + s] = reinterpret_cast<const double*>(e.raw_x[s]);
            } else {  // another process: CUDA IPC (NVLink peer mappings between GPUs)
                void* p = nullptr;
                FG_CUDA(cudaIpcOpenMemHandle(&p, e.h_flags, cudaIpcMemLazyEnablePeerAccess));
                h->opened.push_back(p);
                pflags[q] = static_cast<long long*>(p);
                FG_CUDA(cudaIpcOpenMemHandle(&p, e.h_recv, cudaIpcMemLazyEnablePeerAccess));
                h->opened.push_back(p);
                precv[q] = static_cast<double*>(p);
                const bool pulls_from_q = std::find(h->pull_peers.begin(), h->pull_peers.end(), q) != h->pull_peers.end();
                for (int s = 0; s < e.n_x && pulls_from_q; ++s) {
                    FG_CUDA(cudaIpcOpenMemHandle(&p, e.h_x[s], cudaIpcMemLazyEnablePeerAccess));
                    h->opened.push_back(p);
                    px[static_cast<size_t>(q) * kMaxSpaces + s] = static_cast<const double*>(p);
                }
            }
            // my segment in q's receive buffer
            for (size_t i = 0; i < h->push_row.size(); ++i)
                if (h->push_peer[i] == q) push_off[i] = e.recv_off[me] + h->push_local_idx[i];
        }
        // device CG buffers (femgpu_halo_cg) allocated here, while every rank is in this collective:
        // a cudaMalloc later could wait on the device behind a peer's spinning exchange kernel
        {
            femgpu::Instance& I = *h->inst;
            const long long n = I.output_size;
            std::vector<unsigned char> owned(static_cast<size_t>(n), 1);
            for (int r : h->push_row) owned[static_cast<size_t>(r)] = 0;
            h->d_owned = dev_copy(owned, h->keep);
            for (int k = 0; k < 3; ++k) h->cg_work.push_back(I.alloc<double>(static_cast<size_t>(n)));
            h->cg_work.push_back(I.alloc<double>(kCgBlocks + 8));
        }
        h->d_peer_flags = dev_copy(pflags, h->keep);
        h->d_peer_recv = dev_copy(precv, h->keep);
        h->d_peer_x = dev_copy(px, h->keep);
        h->d_peer_slot = dev_copy(pslot, h->keep);
        h->d_push_off = dev_copy(push_off, h->keep);
        h->imported = true;
    });
}

femgpu_status femgpu_halo_action(femgpu_halo* h, const femgpu_schedule* s, double* y_dev, void* stream) {
    return femgpu::abi_guard([&] {
        if (!h || !h->imported) femgpu::invalid("halo: not imported");
        femgpu::Instance& I = *h->inst;
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        halo_step(*h, kp, y_dev ? y_dev : I.d_y, stream ? static_cast<cudaStream_t>(stream) : I.stream);
    });
}

femgpu_status femgpu_halo_time_steps(femgpu_halo* h, const femgpu_schedule* s, int32_t steps, double* seconds) {
    return femgpu::abi_guard([&] {
        if (!h || !h->imported || steps < 1 || !seconds) femgpu::invalid("halo: not imported / bad arguments");
        femgpu::Instance& I = *h->inst;
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        // stream (not device) synchronisation: ranks sharing a device in one process must not
        // wait on each other's spinning exchange kernels from the host
        FG_CUDA(cudaStreamSynchronize(I.stream));
        FG_CUDA(cudaStreamSynchronize(h->side));
        // one step captured as a CUDA graph (its step numbers live on the device), replayed per step:
        // one graph launch per action instead of six launches (FEMGPU_HALO_GRAPH=0: direct launches)
        const char* ge = std::getenv("FEMGPU_HALO_GRAPH");
        const bool use_graph = !(ge && std::strcmp(ge, "0") == 0);
        cudaGraphExec_t exec = nullptr;
        if (use_graph) {
            cudaGraph_t graph = nullptr;
            FG_CUDA(cudaStreamBeginCapture(I.stream, cudaStreamCaptureModeThreadLocal));
            halo_step(*h, kp, I.d_y, I.stream);
            FG_CUDA(cudaStreamEndCapture(I.stream, &graph));
            FG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
            cudaGraphDestroy(graph);
            --h->step;  // capture did not run a step
        }
        FG_CUDA(cudaEventRecord(I.ev0, I.stream));
        for (int i = 0; i < steps; ++i) {
            if (exec) {
                FG_CUDA(cudaGraphLaunch(exec, I.stream));
                ++h->step;
            } else {
                halo_step(*h, kp, I.d_y, I.stream);
            }
        }
        FG_CUDA(cudaEventRecord(I.ev1, I.stream));
        FG_CUDA(cudaEventSynchronize(I.ev1));
        float ms = 0.f;
        FG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
        if (exec) cudaGraphExecDestroy(exec);
        *seconds = ms * 1e-3;
    });
}

femgpu_status femgpu_halo_cg(femgpu_halo* h, const femgpu_schedule* s, const double* b_dev, double* x_dev, double rtol,
                             int32_t maxiter, int32_t check_every, int32_t* iterations, double* rel_residual) {
    return femgpu::abi_guard([&] {
        if (!h || !h->imported) femgpu::invalid("halo: not imported");
        if (!b_dev || !x_dev) femgpu::invalid("halo_cg: null vector");
        femgpu::Instance& I = *h->inst;
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        if (I.sspaces.size() != 1 || !I.vspaces.empty() || I.sspaces[0].global != I.output_size)
            femgpu::invalid("halo_cg: one scalar trial space numbered like the test space required");
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        const long long n = I.output_size;
        cudaStream_t st = I.stream;
        if (check_every < 1) check_every = 1;
        double *r = h->cg_work[0], *p = h->cg_work[1], *ap = h->cg_work[2], *part = h->cg_work[3];
        double* sc = part + kCgBlocks;  // [0] local, [1] b.b, [2] p.Ap, [3]/[4] r.r alternating
        double* xin = I.sspaces[0].d_x;  // the instance input the exchange pulls from and into
        const dim3 g(kCgBlocks), t(kCgThreads);
        auto allreduce = [&](const double* in, double* out) {
            allreduce_kernel<<<1, 1, 0, st>>>(h->d_peer_flags, h->flags, h->rank, h->world, in, out, ++h->red_epoch,
                                              h->timeout_ns);
            FG_CUDA(cudaGetLastError());
        };
        auto apply = [&](const double* v, double* out) {  // out = A v (owned rows), ghost rows zero
            FG_CUDA(cudaMemcpyAsync(xin, v, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice, st));
            halo_step(*h, kp, out, st);
            cg_mask<<<g, t, 0, st>>>(out, h->d_owned, n);
        };
        apply(x_dev, ap);
        cg_init<<<g, t, 0, st>>>(r, p, b_dev, ap, h->d_owned, n);
        cg_mask_dot<<<g, t, 0, st>>>(b_dev, b_dev, h->d_owned, n, part);
        cg_final<<<1, t, 0, st>>>(part, sc);
        allreduce(sc, sc + 1);
        cg_mask_dot<<<g, t, 0, st>>>(r, r, h->d_owned, n, part);
        cg_final<<<1, t, 0, st>>>(part, sc);
        allreduce(sc, sc + 3);
        double host[5];
        FG_CUDA(cudaMemcpyAsync(host, sc, sizeof host, cudaMemcpyDeviceToHost, st));
        FG_CUDA(cudaStreamSynchronize(st));  // this rank's stream only: peers' kernels may still spin
        const double bnorm = std::sqrt(host[1]);
        double res = std::sqrt(host[3]);
        int it = 0, cur = 3;
        while (res > rtol * bnorm && it < maxiter) {
            apply(p, ap);
            cg_mask_dot<<<g, t, 0, st>>>(p, ap, h->d_owned, n, part);
            cg_final<<<1, t, 0, st>>>(part, sc);
            allreduce(sc, sc + 2);
            cg_update_xr<<<g, t, 0, st>>>(x_dev, r, p, ap, h->d_owned, n, sc + cur, sc + 2, part);
            cg_final<<<1, t, 0, st>>>(part, sc);
            allreduce(sc, sc + (7 - cur));
            cg_update_p<<<g, t, 0, st>>>(p, r, n, sc + (7 - cur), sc + cur);
            FG_CUDA(cudaGetLastError());
            cur = 7 - cur;
            ++it;
            if (it % check_every == 0 || it == maxiter) {
                long long err = 0;
                FG_CUDA(cudaMemcpyAsync(host, sc + cur, sizeof(double), cudaMemcpyDeviceToHost, st));
                FG_CUDA(cudaMemcpyAsync(&err, h->flags + 2, sizeof err, cudaMemcpyDeviceToHost, st));
                FG_CUDA(cudaStreamSynchronize(st));
                res = std::sqrt(host[0]);
                if (err || !std::isfinite(res)) break;  // a timed-out exchange: femgpu_halo_check reports it
            }
        }
        if (iterations) *iterations = it;
        if (rel_residual) *rel_residual = bnorm > 0 ? res / bnorm : res;
    });
}

femgpu_status femgpu_halo_check(femgpu_halo* h, void* stream) {
    return femgpu::abi_guard([&] {
        if (!h) femgpu::invalid("halo: null handle");
        FG_CUDA(cudaSetDevice(h->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->inst->stream;
        long long err[4] = {0, 0, 0, 0};
        FG_CUDA(cudaStreamSynchronize(h->side));
        FG_CUDA(cudaMemcpyAsync(err, h->flags + 2, sizeof err, cudaMemcpyDeviceToHost, s));
        FG_CUDA(cudaStreamSynchronize(s));
        if (err[0]) {
            const char* what = (err[0] & 1) ? "pull" : (err[0] & 2) ? "push" : (err[0] & 4) ? "receive" : "all-reduce";
            femgpu::fail(FEMGPU_E_CUDA, std::string("halo: a peer did not reach the exchange in time (rank ") +
                                            std::to_string(h->rank) + ", step " + std::to_string(h->step) + ": " + what +
                                            " wait on rank " + std::to_string(err[1]) + " saw " + std::to_string(err[2]) +
                                            ", wanted " + std::to_string(err[3]) + ")");
        }
    });
}

}  // extern "C"
