// multi.cu — row-sharded multi-GPU SGEMM (BASELINE.json north_star,
// "Multi-GPU: large problems are partitioned ... by C row-blocks. B is
// broadcast and C is optionally all-gathered with NCCL over NVLink, with
// compute overlapped on streams").
//
// The paper's only distributed use of its SGEMM is the 196-CPU neural-network
// run with no communication details; this is the B200
// design of SURVEY.md §8(e) / §8(f)-2: each rank owns a block of rows of
// op(A) and C, B is broadcast from `root` in column panels, and the GEMM of
// panel c waits only for panel c, so the transfer of later panels overlaps
// the math of earlier ones.
//
// Two data planes for the exchange steps:
//  * NCCL (buffers not registered): ncclBroadcast per B panel on a
//    communication stream; C all-gather as grouped broadcasts into a staging
//    buffer + unpack (KN6).
//  * Copy engines + flags (buffers registered with emm_comm_register_input /
//    _output): B is forwarded along the ring that starts at `root` (root ->
//    root+1 -> ... -> root-1) in chunks of <= 64 MB by cudaMemcpyAsync into
//    the next rank's (IPC-mapped) B buffer — peer copies run on the copy
//    engines, so they take no SMs from the persistent GEMM — each chunk
//    followed by a release store of the call's epoch into the receiver's flag
//    word; the receiver's GEMM of a panel waits (acquire) for the flag of the
//    panel's last chunk.  Every rank sends B once (a pipelined chain uses each
//    GPU's NVLink egress once, the bandwidth optimum of a broadcast through a
//    switch).  C is gathered by the GEMM epilogue storing each finished tile
//    into every rank's C_full (tensor-core modes) or by peer 2-D copies
//    (other modes); a flag per rank closes the call.  Buffers are reused
//    across calls through a "consumed" flag: a rank pushes call e only after
//    its successor has finished reading call e-1.
//
// The same code also runs P VIRTUAL ranks on one GPU
// (emm_debug_comm_create_local): distinct buffers on one device instead of
// IPC-mapped peers, and — since kernels on one GPU must never spin on each
// other — the signal / wait points as CUDA events, all ranks' work enqueued
// in dependency order once the last rank has called.  The harness the tests
// use to drive the P > 1 paths of emm_sgemm_multi on a single B200.
//
// NCCL is loaded at run time (dlopen of the process's libnccl.so.2, normally
// the one torch already loaded), so the library has no link-time NCCL
// dependency and the host-only entry points work on machines without it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "emm_internal.h"

namespace emm {
namespace {

struct Nccl {
    bool ok = false;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclCommGetAsyncError) getAsyncError = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
};

Nccl &nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
        n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
        n.getAsyncError = (decltype(n.getAsyncError))dlsym(h, "ncclCommGetAsyncError");
        n.broadcast = (decltype(n.broadcast))dlsym(h, "ncclBroadcast");
        n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
        n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
        n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
        n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.getAsyncError && n.broadcast && n.groupStart &&
               n.groupEnd && n.allGather;
    });
    return n;
}

constexpr int MAXR = 8;
// flag words per rank (device memory, uint32, monotonically increasing epochs)
constexpr int FL_BREADY = 0;                 // [FL_NCHUNK] B chunk j of this call landed here
constexpr int FL_NCHUNK = 1024;
constexpr int FL_CONSUMED = FL_NCHUNK;       // successor finished reading its B (written by the successor)
constexpr int FL_DONE = FL_NCHUNK + 32;      // [MAXR] rank r finished storing its rows into this C_full
constexpr int FL_WORDS = FL_NCHUNK + 64;
constexpr size_t CHUNK_BYTES = 64u << 20;    // B forwarding granularity

// P virtual ranks on one device (emm_debug_comm_create_local): the tables
// the IPC exchange fills in the multi-process case.
// Arguments of one emm_sgemm_multi call (kept by virtual ranks until the
// last rank of the world has called, see emm_sgemm_multi).
struct MultiArgs {
    char transA, transB;
    int64_t M, N, K;
    float alpha;
    const float *A_local;
    int64_t lda;
    float *B;
    int64_t ldb;
    int root;
    float beta;
    float *C_local;
    int64_t ldc;
    float *C_full;
    int64_t ldc_full;
    cudaStream_t s;
    emm_math_t math;
};

struct Comm;
struct World {
    int nranks = 0;
    std::mutex mu;
    int alive = 0;
    std::vector<cudaEvent_t> ev[MAXR];   // per rank: the signal slots as events
    MultiArgs pending[MAXR] = {};         // per rank: the call waiting for the others
    Comm *pending_comm[MAXR] = {};
    int arrived = 0;
    uint32_t *flags[MAXR] = {};
    float *in[MAXR] = {};
    size_t in_bytes[MAXR] = {};
    float *out[MAXR] = {};
    int64_t out_ld[MAXR] = {};
};

struct Comm {
    ncclComm_t nc = nullptr;               // NCCL mode
    std::shared_ptr<World> world;          // local (virtual-rank) mode
    int nranks = 0, rank = 0, dev = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> evs;
    float *stage = nullptr;  // NCCL all-gather staging (grown on demand)
    size_t stage_bytes = 0;
    void *ws = nullptr;      // tensor-core workspace: A planes | B panel planes | control block
    size_t ws_bytes = 0;
    uint32_t epoch = 0;      // calls of emm_sgemm_multi (identical on every rank)
    // flag words: own array and every peer's (IPC-mapped; own = flags)
    uint32_t *flags = nullptr;
    uint32_t *peer_flags[MAXR] = {};
    bool ce_ok = true;   // peers' flag words mapped (copy-engine data plane possible; same on every rank)
    void *flags_opened[MAXR] = {};
    // registered input (B receive buffer) and the successor's, mapped
    float *in_local = nullptr;
    size_t in_bytes = 0;
    float *in_succ = nullptr;
    void *in_opened = nullptr;
    // registered output: every rank's full C
    float *out_local = nullptr;
    int64_t out_ld = 0;
    float *out_peer[MAXR] = {};
    void *out_opened[MAXR] = {};
    bool local() const { return world != nullptr; }
};

// driver cuMemGetAddressRange (allocation base of a device pointer)
typedef CUresult (*PFN_range)(CUdeviceptr *, size_t *, CUdeviceptr);
PFN_range range_fn() {
    static PFN_range fn = [] {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return (PFN_range)p;
        return (PFN_range) nullptr;
    }();
    return fn;
}

struct IpcBlob {
    cudaIpcMemHandle_t h;
    int64_t offset;   // bytes from the allocation base to the registered pointer
    int64_t a, b;     // ld / size, checked for consistency
    int64_t st;       // the sender's local status (0: the handle is valid)
};

int nccl_status(ncclResult_t r) { return r == ncclSuccess ? 0 : EMM_ERR_NCCL_BASE + (int)r; }
int cuda_st(cudaError_t e) { return e == cudaSuccess ? 0 : EMM_ERR_CUDA_BASE + (int)e; }

int grow(void **p, size_t *have, size_t need) {
    if (*have >= need && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) return EMM_ERR_CUDA_BASE + (int)e;
    *have = need;
    return 0;
}

cudaEvent_t ev_at(Comm *c, size_t i) {
    while (c->evs.size() <= i) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        c->evs.push_back(e);
    }
    return c->evs[i];
}

// IPC handle of the allocation holding `p` (+ offset), all-gathered over NCCL.
// Every rank takes part in the exchange even when its own handle could not be
// made (its blob then carries the failure), so a local error never leaves the
// other ranks waiting in the collective; the result is uniform: 0 on every
// rank, or an error on every rank.
int ipc_allgather(Comm *c, const void *p, int64_t a, int64_t b, std::vector<IpcBlob> &all) {
    Nccl &n = nccl();
    auto rf = range_fn();
    CUdeviceptr base = 0;
    size_t size = 0;
    IpcBlob mine{};
    int lst = (!rf || rf(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) ? EMM_ERR_COMM : 0;
    if (!lst) lst = cuda_st(cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void *>(base)));
    mine.offset = (int64_t)(reinterpret_cast<CUdeviceptr>(p) - base);
    mine.a = a;
    mine.b = b;
    mine.st = lst;
    IpcBlob *dev = nullptr;
    int st = cuda_st(cudaMalloc(&dev, sizeof(IpcBlob) * (c->nranks + 1)));
    if (st) return st;   // no buffer to take part with (device out of memory)
    all.assign(c->nranks, IpcBlob{});
    st = cuda_st(cudaMemcpy(dev + c->nranks, &mine, sizeof mine, cudaMemcpyHostToDevice));
    if (!st) st = nccl_status(n.allGather(dev + c->nranks, dev, sizeof(IpcBlob), ncclUint8, c->nc, c->comm_stream));
    if (!st) st = cuda_st(cudaStreamSynchronize(c->comm_stream));
    if (!st) st = cuda_st(cudaMemcpy(all.data(), dev, sizeof(IpcBlob) * c->nranks, cudaMemcpyDeviceToHost));
    cudaFree(dev);
    if (st) return st;
    for (const IpcBlob &x : all)   // (own blob included: the same code on every rank)
        if (x.st) return EMM_ERR_COMM;   // some rank could not export its buffer
    return 0;
}

// Collective agreement on a registration's outcome: every rank contributes
// its local status (e.g. of opening the peers' handles) and returns the same
// verdict (0 only if every rank succeeded).
int agree(Comm *c, int lst) {
    if (c->nranks == 1) return lst;
    Nccl &n = nccl();
    int64_t *dev = nullptr;
    int st = cuda_st(cudaMalloc(&dev, sizeof(int64_t) * (c->nranks + 1)));
    if (st) return st;
    const int64_t mine = lst;
    std::vector<int64_t> all(c->nranks, 0);
    st = cuda_st(cudaMemcpy(dev + c->nranks, &mine, sizeof mine, cudaMemcpyHostToDevice));
    if (!st) st = nccl_status(n.allGather(dev + c->nranks, dev, sizeof(int64_t), ncclUint8, c->nc, c->comm_stream));
    if (!st) st = cuda_st(cudaStreamSynchronize(c->comm_stream));
    if (!st) st = cuda_st(cudaMemcpy(all.data(), dev, sizeof(int64_t) * c->nranks, cudaMemcpyDeviceToHost));
    cudaFree(dev);
    if (st) return st;
    for (int64_t x : all)   // (own status included: the same code on every rank)
        if (x) return EMM_ERR_COMM;
    return 0;
}

int ipc_open(const IpcBlob &b, void **opened, void **ptr) {
    void *p = nullptr;
    int st = cuda_st(cudaIpcOpenMemHandle(&p, b.h, cudaIpcMemLazyEnablePeerAccess));
    if (st) return st;
    *opened = p;
    *ptr = static_cast<uint8_t *>(p) + b.offset;
    return 0;
}

// ---------------------------------------------------------------- flag kernels
// Release store of the epoch into a (possibly peer) flag word, after every
// earlier operation of the stream (copies, GEMMs and their peer stores).
struct FlagSet {
    uint32_t *f[MAXR];
    int n;
};
__global__ void flag_set_kernel(const FlagSet fs, uint32_t v) {
    if (threadIdx.x < fs.n) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(fs.f[threadIdx.x]), "r"(v) : "memory");
    }
}
// Acquire-spin until every word of f[idx[i]] reaches the epoch (wrap-safe
// compare).  Bounded: traps after ~20 s so a protocol error cannot wedge
// the GPU.
struct FlagWait {
    const uint32_t *f[MAXR];
    int n;
};
__global__ void flag_wait_kernel(const FlagWait fw, uint32_t v) {
    if (threadIdx.x >= fw.n) return;
    const long long t0 = clock64();
    while (true) {
        uint32_t x;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(fw.f[threadIdx.x]) : "memory");
        if ((int32_t)(x - v) >= 0) break;
        __nanosleep(256);
        if (clock64() - t0 > 40000000000LL) __trap();
    }
}

cudaError_t flag_set(uint32_t *const *fs, int n, uint32_t v, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    FlagSet a{};
    for (int i = 0; i < n; ++i) a.f[i] = fs[i];
    a.n = n;
    flag_set_kernel<<<1, 32, 0, s>>>(a, v);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}
cudaError_t flag_wait(const uint32_t *const *fs, int n, uint32_t v, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    FlagWait a{};
    for (int i = 0; i < n; ++i) a.f[i] = fs[i];
    a.n = n;
    flag_wait_kernel<<<1, 32, 0, s>>>(a, v);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

int comm_init_streams(Comm *c) {
    int st = cuda_st(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    if (!st) st = cuda_st(cudaMalloc(&c->flags, FL_WORDS * sizeof(uint32_t)));
    if (!st) st = cuda_st(cudaMemset(c->flags, 0, FL_WORDS * sizeof(uint32_t)));
    if (!st) st = cuda_st(cudaDeviceSynchronize());
    return st;
}

// peer flag arrays: mapped by IPC (NCCL mode) or taken from the world table
int resolve_flags(Comm *c) {
    if (c->nranks == 1 || c->peer_flags[(c->rank + 1) % c->nranks]) return 0;
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        for (int r = 0; r < c->nranks; ++r) {
            if (!c->world->flags[r]) return EMM_ERR_COMM;
            c->peer_flags[r] = c->world->flags[r];
        }
        return 0;
    }
    return EMM_ERR_COMM;   // NCCL mode maps them in emm_comm_create
}

}  // namespace
}  // namespace emm

using namespace emm;

extern "C" int64_t emm_multi_panel_cols(int64_t N) {
    // 4 panels, each >= 1024 columns and a multiple of the 256-wide tile: the
    // first panel's broadcast is exposed (~1/4 of B), the others hide under
    // the previous panel's GEMM; wider panels keep each panel GEMM at many
    // full waves (c5 at P=8: 16 x 32 = 512 tiles = 6.9 waves of 74 CTA pairs,
    // vs 3.5 waves with 8 panels).
    int64_t panel = (N + 3) / 4;
    if (panel < 1024) panel = 1024;
    return (panel + 255) / 256 * 256;
}

extern "C" int emm_get_unique_id(void *id128) {
    Nccl &n = nccl();
    if (!n.ok || !id128) return EMM_ERR_COMM;
    ncclUniqueId id;
    int st = nccl_status(n.getUniqueId(&id));
    if (!st) memcpy(id128, &id, sizeof id);
    return st;
}

extern "C" int emm_comm_create(void **comm, const void *id128, int nranks, int rank) {
    Nccl &n = nccl();
    if (!n.ok || !comm || !id128 || nranks < 1 || nranks > MAXR || rank < 0 || rank >= nranks) return EMM_ERR_COMM;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    Comm *c = new Comm();
    c->nranks = nranks;
    c->rank = rank;
    cudaGetDevice(&c->dev);
    int st = nccl_status(n.commInitRank(&c->nc, nranks, id, rank));
    if (!st) st = comm_init_streams(c);
    // map every peer's flag words (copy-engine data plane)
    if (!st && nranks > 1) {
        std::vector<IpcBlob> all;
        st = ipc_allgather(c, c->flags, FL_WORDS, 0, all);
        if (!st) {   // (an exchange error is uniform; an open error is agreed below)
            int ost = 0;
            for (int r = 0; r < nranks && !ost; ++r) {
                if (r == rank) {
                    c->peer_flags[r] = c->flags;
                    continue;
                }
                void *p = nullptr;
                ost = ipc_open(all[r], &c->flags_opened[r], &p);
                c->peer_flags[r] = static_cast<uint32_t *>(p);
            }
            st = agree(c, ost);
        }
        if (st && st != EMM_ERR_COMM) {
            // (NCCL / CUDA failure of the exchange itself: the communicator is unusable)
        } else if (st) {
            // some rank cannot map its peers' memory (no CUDA IPC / P2P): every
            // rank keeps the communicator for the NCCL data plane only; the
            // registrations of the copy-engine plane then fail on every rank
            for (int r = 0; r < nranks; ++r) {
                if (c->flags_opened[r]) cudaIpcCloseMemHandle(c->flags_opened[r]);
                c->flags_opened[r] = nullptr;
                c->peer_flags[r] = nullptr;
            }
            c->ce_ok = false;
            st = 0;
        }
    } else if (!st) {
        c->peer_flags[0] = c->flags;
    }
    if (st) {
        emm_comm_destroy(c);
        return st;
    }
    *comm = c;
    return 0;
}

// P virtual ranks on the current device (tests): comms[r] is rank r of a
// world whose exchange steps are device copies + flags between distinct
// buffers on this one GPU (no NCCL).  Every rank must then register its B
// buffer (emm_comm_register_input) and, for a gathered output, its C_full.
extern "C" int emm_debug_comm_create_local(int nranks, void **comms) {
    if (!comms || nranks < 1 || nranks > MAXR) return EMM_ERR_COMM;
    auto w = std::make_shared<World>();
    w->nranks = nranks;
    for (int r = 0; r < nranks; ++r) comms[r] = nullptr;
    for (int r = 0; r < nranks; ++r) {
        Comm *c = new Comm();
        c->nranks = nranks;
        c->rank = r;
        c->world = w;
        cudaGetDevice(&c->dev);
        int st = comm_init_streams(c);
        if (st) {
            delete c;
            for (int q = 0; q < r; ++q) emm_comm_destroy(comms[q]);
            return st;
        }
        w->flags[r] = c->flags;
        comms[r] = c;
    }
    w->alive = nranks;
    return 0;
}

extern "C" int emm_comm_unregister_output(void *comm) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    cudaStreamSynchronize(c->comm_stream);
    for (int r = 0; r < MAXR; ++r) {
        if (c->out_opened[r]) cudaIpcCloseMemHandle(c->out_opened[r]);
        c->out_opened[r] = nullptr;
        c->out_peer[r] = nullptr;
    }
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        c->world->out[c->rank] = nullptr;
    }
    c->out_local = nullptr;
    c->out_ld = 0;
    return 0;
}

// Collective: every rank registers its M x N (ld_full) full-output buffer;
// the peers' buffers are mapped (CUDA IPC handles all-gathered over NCCL),
// so emm_sgemm_multi can store C tiles straight into them from the GEMM
// epilogue (NVLink peer stores, no all-gather launch).
extern "C" int emm_comm_register_output(void *comm, float *C_full, int64_t ld_full) {
    if (!comm || !C_full || ld_full < 1) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    emm_comm_unregister_output(comm);
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        c->world->out[c->rank] = C_full;
        c->world->out_ld[c->rank] = ld_full;
        c->out_local = C_full;
        c->out_ld = ld_full;
        return 0;   // peers resolved at call time (registration order is free)
    }
    if (!nccl().ok || !c->ce_ok) return EMM_ERR_COMM;
    std::vector<IpcBlob> all;
    int st = c->nranks > 1 ? ipc_allgather(c, C_full, ld_full, 0, all) : 0;
    if (!st && c->nranks > 1) {
        int ost = 0;
        for (int r = 0; r < c->nranks && !ost; ++r) {
            if (r == c->rank) {
                c->out_peer[r] = C_full;
                continue;
            }
            if (all[r].a != ld_full) ost = EMM_ERR_COMM;   // identical layouts required
            void *p = nullptr;
            if (!ost) ost = ipc_open(all[r], &c->out_opened[r], &p);
            c->out_peer[r] = static_cast<float *>(p);
        }
        st = agree(c, ost);
    } else if (!st) {
        c->out_peer[0] = C_full;
    }
    if (st) {
        emm_comm_unregister_output(comm);
        return st;
    }
    c->out_local = C_full;
    c->out_ld = ld_full;
    return 0;
}

extern "C" int emm_comm_unregister_input(void *comm) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    cudaStreamSynchronize(c->comm_stream);
    if (c->in_opened) cudaIpcCloseMemHandle(c->in_opened);
    c->in_opened = nullptr;
    c->in_succ = nullptr;
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        c->world->in[c->rank] = nullptr;
    }
    c->in_local = nullptr;
    c->in_bytes = 0;
    return 0;
}

// Collective: register this rank's B buffer (root: the source; others: the
// receive buffer) of `bytes` bytes.  emm_sgemm_multi with that B then
// forwards B along the ring by peer copies on the copy engines.
extern "C" int emm_comm_register_input(void *comm, float *B, size_t bytes) {
    if (!comm || !B || bytes == 0) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    emm_comm_unregister_input(comm);
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        c->world->in[c->rank] = B;
        c->world->in_bytes[c->rank] = bytes;
        c->in_local = B;
        c->in_bytes = bytes;
        return 0;
    }
    if (!nccl().ok || !c->ce_ok) return EMM_ERR_COMM;
    int st = 0;
    if (c->nranks > 1) {
        std::vector<IpcBlob> all;
        st = ipc_allgather(c, B, 0, (int64_t)bytes, all);
        if (!st) {
            const int succ = (c->rank + 1) % c->nranks;
            int ost = 0;
            for (int r = 0; r < c->nranks && !ost; ++r)
                if ((size_t)all[r].b != bytes) ost = EMM_ERR_COMM;
            void *p = nullptr;
            if (!ost) ost = ipc_open(all[succ], &c->in_opened, &p);
            c->in_succ = static_cast<float *>(p);
            st = agree(c, ost);
        }
    }
    if (st) {
        emm_comm_unregister_input(comm);
        return st;
    }
    c->in_local = B;
    c->in_bytes = bytes;
    return 0;
}

extern "C" int emm_comm_destroy(void *comm) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    emm_comm_unregister_output(comm);
    emm_comm_unregister_input(comm);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    for (int r = 0; r < MAXR; ++r)
        if (c->flags_opened[r]) cudaIpcCloseMemHandle(c->flags_opened[r]);
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        c->world->flags[c->rank] = nullptr;
        for (auto e : c->world->ev[c->rank]) cudaEventDestroy(e);
        c->world->ev[c->rank].clear();
        c->world->pending_comm[c->rank] = nullptr;
    }
    if (c->flags) cudaFree(c->flags);
    for (auto e : c->evs) cudaEventDestroy(e);
    if (c->stage) cudaFree(c->stage);
    if (c->ws) cudaFree(c->ws);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    int st = 0;
    if (c->nc) st = nccl_status(nccl().commDestroy(c->nc));
    delete c;
    return st;
}

// B chunks of one call: [panel p] = chunks [pc[p], pc[p+1]); chunk j covers
// bytes [off[j], off[j+1]) of B.
struct Chunks {
    std::vector<int64_t> pc;
    std::vector<size_t> off;
};
// transB = 'N': whole columns per chunk (<= CHUNK_BYTES unless one column is
// larger), chunk boundaries at every panel boundary; 'T': one panel of byte
// chunks.  The chunk size doubles until the count fits the flag words.
static Chunks make_chunks(bool bN, int64_t N, int64_t K, int64_t panel) {
    const size_t col_bytes = (size_t)K * 4;
    const size_t total = (size_t)N * K * 4;
    for (size_t chunk = CHUNK_BYTES;; chunk *= 2) {
        Chunks ch;
        ch.off.push_back(0);
        ch.pc.push_back(0);
        if (bN) {
            const int64_t cols_per = col_bytes > 0 ? std::max<int64_t>(1, (int64_t)(chunk / col_bytes)) : N;
            for (int64_t c0 = 0; c0 < N; c0 += panel) {
                const int64_t c1 = std::min(N, c0 + panel);
                for (int64_t x = c0; x < c1; x += cols_per)
                    ch.off.push_back((size_t)std::min(c1, x + cols_per) * col_bytes);
                ch.pc.push_back((int64_t)ch.off.size() - 1);
            }
        } else {
            for (size_t o = 0; o < total; o += chunk) ch.off.push_back(std::min(total, o + chunk));
            ch.pc.push_back((int64_t)ch.off.size() - 1);
        }
        if ((int64_t)ch.off.size() - 1 <= FL_NCHUNK) return ch;
    }
}

// Host replay of the B chunk plan (tests): chunk byte offsets off[0..n] in
// out_off (n + 1 entries) and, per panel p, the index of its first chunk in
// out_pc (npanel + 1 entries).  Returns n, or -1 if a buffer is too small.
extern "C" int emm_debug_ring_chunks(int64_t N, int64_t K, char transB, int64_t *out_off, int cap_off,
                                     int64_t *out_pc, int cap_pc) {
    const bool bN = transB == 'N' || transB == 'n';
    const Chunks ch = make_chunks(bN, N, K, bN ? emm_multi_panel_cols(N) : N);
    if ((int)ch.off.size() > cap_off || (int)ch.pc.size() > cap_pc) return -1;
    for (size_t i = 0; i < ch.off.size(); ++i) out_off[i] = (int64_t)ch.off[i];
    for (size_t i = 0; i < ch.pc.size(); ++i) out_pc[i] = ch.pc[i];
    return (int)ch.off.size() - 1;
}

namespace emm {
namespace {

// ---- device-side synchronisation of the copy-engine data plane -----------
// Across GPUs (one process per GPU, IPC-mapped flag words): release-store /
// acquire-spin kernels on the epoch.  Virtual ranks on ONE GPU must not spin
// on each other (nothing guarantees that separately launched kernels run at
// the same time): there the same signal / wait points are CUDA events, and
// the world enqueues all ranks' work in dependency order once every rank has
// called (emm_sgemm_multi).
cudaEvent_t world_event(World *w, int rank, int slot) {
    std::lock_guard<std::mutex> g(w->mu);
    auto &v = w->ev[rank];
    while ((int)v.size() <= slot) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        v.push_back(e);
    }
    return v[slot];
}
// signal slot `slot` of each rank in targets[0..n)
int sync_signal(Comm *c, const int *targets, int n, int slot, uint32_t epoch, cudaStream_t s) {
    if (n <= 0) return 0;
    if (c->local()) {
        for (int i = 0; i < n; ++i) {
            cudaEvent_t e = world_event(c->world.get(), targets[i], slot);
            if (!e) return EMM_ERR_NOMEM;
            int st = cuda_st(cudaEventRecord(e, s));
            if (st) return st;
        }
        return 0;
    }
    uint32_t *fs[MAXR];
    for (int i = 0; i < n; ++i) fs[i] = c->peer_flags[targets[i]] + slot;
    return cuda_st(flag_set(fs, n, epoch, s));
}
// wait for this rank's slots[0..n) to reach the epoch
int sync_wait(Comm *c, const int *slots, int n, uint32_t epoch, cudaStream_t s) {
    if (n <= 0) return 0;
    if (c->local()) {
        for (int i = 0; i < n; ++i) {
            cudaEvent_t e = world_event(c->world.get(), c->rank, slots[i]);
            if (!e) return EMM_ERR_NOMEM;
            int st = cuda_st(cudaStreamWaitEvent(s, e, 0));
            if (st) return st;
        }
        return 0;
    }
    const uint32_t *fw[MAXR];
    for (int i = 0; i < n; ++i) fw[i] = c->flags + slots[i];
    return cuda_st(flag_wait(fw, n, epoch, s));
}

// Everything one rank enqueues for a call, up to (and including) its "done"
// signals; done_wait then completes the gathered output.
int enqueue_main(Comm *c, const MultiArgs &a, bool *done_pending) {
    *done_pending = false;
    const char transA = a.transA, transB = a.transB;
    const int64_t M = a.M, N = a.N, K = a.K;
    const float alpha = a.alpha, beta = a.beta;
    const float *A_local = a.A_local;
    const int64_t lda = a.lda, ldb = a.ldb, ldc = a.ldc, ldc_full = a.ldc_full;
    float *B = a.B, *C_local = a.C_local, *C_full = a.C_full;
    const int root = a.root;
    const emm_math_t math = a.math;
    cudaStream_t s = a.s;
    Nccl &n = nccl();
    const int P = c->nranks;
    const bool bN = (transB == 'N' || transB == 'n');
    int64_t row0 = 0, rows = 0;
    emm_row_partition(M, P, c->rank, &row0, &rows);
    const size_t b_bytes = (size_t)(bN ? K * N : N * K) * 4;
    int st = 0;
    // data plane: copy engines + flags when B (and C_full, if gathered) are
    // registered; NCCL otherwise.  The choice depends only on arguments every
    // rank passes identically (and registrations, which are collective), so
    // all ranks take the same branch.
    const bool ce_in = P > 1 && B == c->in_local && c->in_bytes >= b_bytes && (c->local() || c->in_succ);
    const bool ce_out = C_full && C_full == c->out_local && ldc_full == c->out_ld;
    if (c->local() && P > 1 && (!ce_in || (C_full && !ce_out))) return EMM_ERR_COMM;   // no NCCL to fall back on
    if ((ce_in || (ce_out && P > 1)) && (st = resolve_flags(c))) return st;
    float *in_succ = c->in_succ;
    float *out_peer[MAXR] = {};
    for (int r = 0; r < P; ++r) out_peer[r] = c->out_peer[r];
    if (c->local()) {
        std::lock_guard<std::mutex> g(c->world->mu);
        in_succ = c->world->in[(c->rank + 1) % P];
        if (ce_in && (!in_succ || c->world->in_bytes[(c->rank + 1) % P] < b_bytes)) return EMM_ERR_COMM;
        if (ce_out)
            for (int r = 0; r < P; ++r) {
                out_peer[r] = c->world->out[r];
                if (!out_peer[r] || c->world->out_ld[r] != ldc_full) return EMM_ERR_COMM;
            }
    } else if (ce_out) {
        out_peer[c->rank] = c->out_local;
    }
    const uint32_t epoch = ++c->epoch;   // identical on every rank (collective call order)
    const int pos = (c->rank - root + P) % P;       // position in the ring that starts at root
    const int succ = (c->rank + 1) % P, pred = (c->rank - 1 + P) % P;
    const bool has_succ = pos < P - 1, has_pred = pos > 0;

    // Gate the communication stream on the caller's stream (B / C ready;
    // e0 was recorded on it when the call was made).
    st = cuda_st(cudaStreamWaitEvent(c->comm_stream, ev_at(c, 0), 0));
    if (st) return st;

    const int64_t panel = bN ? emm_multi_panel_cols(N) : N;
    // Tensor-core modes: op(A)'s rows are re-buffered ONCE per call into
    // K-major planes in the communicator's cached workspace; each B panel is
    // re-buffered after it arrived and multiplied (one GEMM launch per
    // panel).  FFMA / alpha == 0 / K == 0 / skinny: one emm_sgemm_ex per panel.
    const bool tc = math != EMM_MATH_FFMA && !(alpha == 0.0f || K == 0) && rows > SKINNY_MAX &&
                    N > SKINNY_MAX && 2.0 * rows * (double)N * K > (double)(1 << 24);
    const int terms = math == EMM_MATH_3XTF32 ? 3 : math == EMM_MATH_TF32_BF16 ? 2 : 1;
    const int planes = terms >= 2 ? 2 : 1;
    const int pmode = math == EMM_MATH_3XTF32 ? PK_FULL3_ : math == EMM_MATH_TF32_BF16 ? PK_FULLX_ : PK_FULL1_;
    const int64_t Kp = tc_kpad(K);
    float *Ap = nullptr, *Bp = nullptr;
    unsigned int *ctrl = nullptr;
    // 3xTF32 on TMA-legal operands: KN1X reads op(A)'s rows and each B panel
    // in place (no re-buffering, the split in the kernel) — emm_sgemm_ex's
    // default; otherwise op(A) re-buffered once and each panel after arrival
    const bool xs = tc && terms == 3 && tc_prefer_xs(rows, N, K) && tma_legal(A_local, lda) && tma_legal(B, ldb);
    if (xs && rows > 0 && N > 0) {
        if ((st = grow(&c->ws, &c->ws_bytes, 1024))) return st;
        ctrl = reinterpret_cast<unsigned int *>(c->ws);
    } else if (tc && rows > 0 && N > 0) {
        const size_t a_bytes = align_up((size_t)planes * rows * Kp * 4, 1024);
        const size_t bp_bytes = align_up((size_t)planes * panel * Kp * 4, 1024);
        // stream-ordered reuse: the previous call's kernels on `s` are ordered before this one
        if ((st = grow(&c->ws, &c->ws_bytes, a_bytes + bp_bytes + 1024))) return st;
        Ap = reinterpret_cast<float *>(c->ws);
        Bp = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(c->ws) + a_bytes);
        ctrl = reinterpret_cast<unsigned int *>(reinterpret_cast<uint8_t *>(c->ws) + a_bytes + bp_bytes);
        PackArgs pa;
        pa.X = A_local; pa.ld = lda; pa.R = rows; pa.kcontig = !(transA == 'N' || transA == 'n');
        pa.out0 = Ap; pa.ld0 = Kp; pa.out1 = Ap + (size_t)rows * Kp; pa.ld1 = Kp; pa.b_side = false;
        st = cuda_st(launch_pack(pmode, pa, nullptr, K, nullptr, s));
    }
    // fused all-gather: C_full was registered -> the GEMM epilogue stores into
    // every rank's C_full directly (tensor-core modes)
    const bool fused = tc && ce_out;
    auto panel_gemm = [&](const float *bp, int64_t nc, float *cp) -> int {
        if (rows == 0 || nc == 0) return 0;
        if (!tc)
            return emm_sgemm_ex(transA, transB, rows, nc, K, alpha, A_local, lda, bp, ldb, beta, cp, ldc, s, math,
                                nullptr, 0);
        PeerOut pe;
        if (fused) {
            pe.n = P;
            for (int r = 0; r < P; ++r) pe.base[r] = out_peer[r];
            pe.ld = ldc_full;
            pe.row_off = row0;
            pe.col_off = (cp - C_local) / ldc;   // the panel's first column
        }
        if (xs) {
            cudaError_t e = cudaMemsetAsync(ctrl, 0, 128, s);   // the panel's wave-lockstep counter
            const TcPlane a0{A_local, lda, transA == 'N' || transA == 'n', K};
            const TcPlane b0{bp, ldb, !bN, K};
            if (e == cudaSuccess)
                e = launch_tc_xs_sgemm(a0, b0, rows, nc, K, alpha, beta, cp, ldc, ctrl, 1, nullptr, s,
                                       fused ? &pe : nullptr);
            return cuda_st(e);
        }
        PackArgs pb;
        pb.X = bp; pb.ld = ldb; pb.R = nc; pb.kcontig = bN;
        pb.out0 = Bp; pb.ld0 = Kp; pb.out1 = Bp + (size_t)nc * Kp; pb.ld1 = Kp; pb.b_side = true;
        cudaError_t e = launch_pack(pmode, pb, nullptr, K, ctrl, s);   // also zeroes the lockstep counter
        TcOperands ops;
        ops.a0 = TcPlane{Ap, Kp, false, Kp};
        ops.b0 = TcPlane{Bp, Kp, false, Kp};
        if (planes == 2) {
            ops.a1 = TcPlane{Ap + (size_t)rows * Kp, Kp, false, Kp};
            ops.b1 = TcPlane{Bp + (size_t)nc * Kp, Kp, false, Kp};
        }
        if (e == cudaSuccess)
            e = launch_tc_sgemm(terms, ops, rows, nc, K, alpha, beta, cp, ldc, ctrl, 1, nullptr, s,
                                fused ? &pe : nullptr);
        return cuda_st(e);
    };

    if (!st && ce_in) {
        // ---- copy-engine ring: forward each chunk to the successor as soon
        // as it is here; the GEMM of panel p waits for its last chunk.
        const Chunks ch = make_chunks(bN, N, K, panel);
        const int nchunk = (int)ch.off.size() - 1;
        if (has_succ) {
            // the successor finished reading the previous call's B
            const int sc = FL_CONSUMED;
            st = sync_wait(c, &sc, 1, epoch - 1, c->comm_stream);
            for (int j = 0; j < nchunk && !st; ++j) {
                if (has_pred) {
                    const int sb = FL_BREADY + j;
                    st = sync_wait(c, &sb, 1, epoch, c->comm_stream);
                }
                const size_t o = ch.off[j], nb = ch.off[j + 1] - o;
                if (!st && nb)
                    st = cuda_st(cudaMemcpyAsync(reinterpret_cast<uint8_t *>(in_succ) + o,
                                                 reinterpret_cast<const uint8_t *>(B) + o, nb,
                                                 cudaMemcpyDeviceToDevice, c->comm_stream));
                if (!st) st = sync_signal(c, &succ, 1, FL_BREADY + j, epoch, c->comm_stream);
            }
        }
        const int npanel = (int)ch.pc.size() - 1;
        for (int p = 0; p < npanel && !st; ++p) {
            if (has_pred && ch.pc[p + 1] > ch.pc[p]) {
                const int sb = FL_BREADY + (int)(ch.pc[p + 1] - 1);
                st = sync_wait(c, &sb, 1, epoch, s);
            }
            if (st) break;
            if (bN) {
                const int64_t c0 = (int64_t)p * panel, nc = std::min(panel, N - c0);
                st = panel_gemm(B + c0 * ldb, nc, C_local + c0 * ldc);
            } else {
                st = panel_gemm(B, N, C_local);
            }
        }
        // every read of this rank's B (GEMMs on s, forwarding on comm_stream)
        // is done -> tell the predecessor it may overwrite it
        cudaEvent_t ef = ev_at(c, 1);
        if (!st && !ef) st = EMM_ERR_NOMEM;
        if (!st) st = cuda_st(cudaEventRecord(ef, c->comm_stream));
        if (!st) st = cuda_st(cudaStreamWaitEvent(s, ef, 0));
        // (always, whatever this call's root: the ring predecessor waits for
        // it before pushing the next call's B, which may start elsewhere)
        if (!st) st = sync_signal(c, &pred, 1, FL_CONSUMED, epoch, s);
    } else if (!st && bN && N > 0) {
        // ---- NCCL: column panels of B, contiguous K x nc ranges; the GEMM of
        // panel c waits only for panel c's broadcast.
        size_t idx = 2;
        for (int64_t c0 = 0; c0 < N && !st; c0 += panel, ++idx) {
            const int64_t nc = (N - c0 < panel) ? N - c0 : panel;
            float *bp = B + c0 * ldb;
            if (K > 0 && P > 1)
                st = nccl_status(n.broadcast(bp, bp, (size_t)(K * nc), ncclFloat32, root, c->nc, c->comm_stream));
            cudaEvent_t ev = ev_at(c, idx);
            if (!st && !ev) st = EMM_ERR_NOMEM;
            if (!st) st = cuda_st(cudaEventRecord(ev, c->comm_stream));
            if (!st) st = cuda_st(cudaStreamWaitEvent(s, ev, 0));
            if (!st) st = panel_gemm(bp, nc, C_local + c0 * ldc);
        }
    } else if (!st && N > 0) {
        // transB = 'T' over NCCL: B's stored columns run along K; broadcast it
        // whole (no panel overlap), then one GEMM.
        if (b_bytes > 0 && P > 1)
            st = nccl_status(n.broadcast(B, B, b_bytes / 4, ncclFloat32, root, c->nc, c->comm_stream));
        cudaEvent_t ev = ev_at(c, 2);
        if (!st) st = cuda_st(cudaEventRecord(ev, c->comm_stream));
        if (!st) st = cuda_st(cudaStreamWaitEvent(s, ev, 0));
        if (!st) st = panel_gemm(B, N, C_local);
    }
    if (st) return st;

    if (C_full && ce_out) {
        // ---- gathered output through the registered peers: the tensor-core
        // epilogue already stored this rank's rows into every C_full (fused);
        // other modes copy them (2-D peer copies, strided column-major rows).
        if (!fused && rows > 0 && N > 0)
            for (int r = 0; r < P && !st; ++r)
                st = cuda_st(cudaMemcpy2DAsync(out_peer[r] + row0, (size_t)ldc_full * 4, C_local, (size_t)ldc * 4,
                                               (size_t)rows * 4, (size_t)N, cudaMemcpyDeviceToDevice, s));
        if (!st && P > 1) {
            // every rank tells every rank its rows are in place (then, in
            // done_wait, waits for all of them: C_full is complete on `s`)
            int targets[MAXR], k = 0;
            for (int r = 0; r < P; ++r)
                if (r != c->rank) targets[k++] = r;
            st = sync_signal(c, targets, k, FL_DONE + c->rank, epoch, s);
            *done_pending = !st;
        }
        return st;
    }
    if (C_full) {
        if (c->local()) return EMM_ERR_COMM;
        // ---- NCCL all-gather of the row blocks: compact own block into the
        // rank-major staging buffer, P broadcasts in one NCCL group, then
        // unpack (KN6).
        const size_t need = (size_t)M * (size_t)N * 4;
        if (c->stage_bytes < need) {
            if (c->stage) cudaFree(c->stage);
            c->stage = nullptr;
            c->stage_bytes = 0;
            if ((st = cuda_st(cudaMalloc(&c->stage, need)))) return st;
            c->stage_bytes = need;
        }
        std::vector<int64_t> r0s(P), rws(P), offs(P);
        int64_t off = 0;
        for (int r = 0; r < P; ++r) {
            emm_row_partition(M, P, r, &r0s[r], &rws[r]);
            offs[r] = off;
            off += rws[r] * N;
        }
        if (rows > 0 && N > 0)
            st = cuda_st(cudaMemcpy2DAsync(c->stage + offs[c->rank], (size_t)rows * 4, C_local, (size_t)ldc * 4,
                                           (size_t)rows * 4, (size_t)N, cudaMemcpyDeviceToDevice, s));
        if (st) return st;
        if (P > 1) {
            n.groupStart();
            for (int r = 0; r < P; ++r)
                if (rws[r] > 0)
                    n.broadcast(c->stage + offs[r], c->stage + offs[r], (size_t)(rws[r] * N), ncclFloat32, r, c->nc,
                                s);
            st = nccl_status(n.groupEnd());
            if (st) return st;
        }
        st = cuda_st(launch_unpack_rows(c->stage, P, r0s.data(), rws.data(), N, C_full, ldc_full, s));
    }
    return st;
}

int done_wait(Comm *c, cudaStream_t s) {
    int slots[MAXR], k = 0;
    for (int r = 0; r < c->nranks; ++r)
        if (r != c->rank) slots[k++] = FL_DONE + r;
    return sync_wait(c, slots, k, c->epoch, s);
}

}  // namespace
}  // namespace emm

extern "C" int emm_sgemm_multi(void *comm, char transA, char transB, int64_t M, int64_t N, int64_t K, float alpha,
                               const float *A_local, int64_t lda, float *B, int64_t ldb, int root, float beta,
                               float *C_local, int64_t ldc, float *C_full, int64_t ldc_full, void *stream,
                               emm_math_t math) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    Nccl &n = nccl();
    if (root < 0 || root >= c->nranks) return EMM_ERR_COMM;
    const int P = c->nranks;
    const bool bN = (transB == 'N' || transB == 'n');
    if (K >= 0 && ldb != (bN ? (K > 1 ? K : 1) : (N > 1 ? N : 1))) return -10;  // panels must be contiguous
    if (!c->local()) {
        if (!n.ok) return EMM_ERR_COMM;
        ncclResult_t async_err = ncclSuccess;
        n.getAsyncError(c->nc, &async_err);
        if (async_err != ncclSuccess) return nccl_status(async_err);
    }
    int64_t row0 = 0, rows = 0;
    emm_row_partition(M, P, c->rank, &row0, &rows);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int st = check_args(transA, transB, rows, N, K, lda, ldb, ldc > 0 ? ldc : 1);
    if (!st) st = check_device();
    if (st) return st;
    if (C_full && ldc_full < (M > 1 ? M : 1)) return -17;
    // the caller's stream gates this call's reads of B / C
    cudaEvent_t e0 = ev_at(c, 0);
    if (!e0) return EMM_ERR_NOMEM;
    if ((st = cuda_st(cudaEventRecord(e0, s)))) return st;
    const MultiArgs args{transA, transB, M, N, K, alpha, A_local, lda, B, ldb, root, beta,
                         C_local, ldc, C_full, ldc_full, s, math};
    if (!c->local() || P == 1) {
        bool dw = false;
        st = enqueue_main(c, args, &dw);
        if (!st && dw) st = done_wait(c, s);
        return st;
    }
    // Virtual ranks: nothing is enqueued until every rank of the world has
    // called; the last caller enqueues all ranks' work in dependency order
    // (the ring from root, then every rank's wait for the others' "done"),
    // so that each event a stream waits on is recorded first.  Earlier calls
    // return 0 (errors surface on the last call); until then a rank's stream
    // must not receive other work.
    World *w = c->world.get();
    std::vector<std::pair<Comm *, MultiArgs>> calls;
    {
        std::lock_guard<std::mutex> g(w->mu);
        w->pending[c->rank] = args;
        w->pending_comm[c->rank] = c;
        if (++w->arrived < P) return 0;
        w->arrived = 0;
        for (int k = 0; k < P; ++k) {
            const int r = (root + k) % P;
            calls.emplace_back(w->pending_comm[r], w->pending[r]);
        }
    }
    bool dw[MAXR] = {};
    for (int k = 0; k < P && !st; ++k) st = enqueue_main(calls[k].first, calls[k].second, &dw[k]);
    for (int k = 0; k < P && !st; ++k)
        if (dw[k]) st = done_wait(calls[k].first, calls[k].second.s);
    return st;
}

