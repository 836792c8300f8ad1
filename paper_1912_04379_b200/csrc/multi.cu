// multi.cu — row-sharded multi-GPU SGEMM over NCCL (BASELINE.json north_star,
// "Multi-GPU: large problems are partitioned ... by C row-blocks. B is
// broadcast and C is optionally all-gathered with NCCL over NVLink, with
// compute overlapped on streams").
//
// The paper's only distributed use of its SGEMM is the 196-CPU neural-network
// run with no communication details; this is the B200
// design of SURVEY.md §8(e): each rank owns a block of rows of op(A) and C,
// B is broadcast from `root` in column panels on a communication stream, and
// the GEMM of panel c (compute stream) waits only for panel c, so the
// transfer of panel c+1 overlaps the math of panel c.
//
// NCCL is loaded at run time (dlopen of the process's libnccl.so.2, normally
// the one torch already loaded), so the library has no link-time NCCL
// dependency and the host-only entry points work on machines without it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
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
    decltype(&ncclAllReduce) allReduce = nullptr;
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
        n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
        n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.getAsyncError && n.broadcast && n.groupStart &&
               n.groupEnd && n.allGather && n.allReduce;
    });
    return n;
}

struct Comm {
    ncclComm_t nc = nullptr;
    int nranks = 0, rank = 0, dev = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> evs;
    float *stage = nullptr;  // all-gather staging (grown on demand)
    size_t stage_bytes = 0;
    void *ws = nullptr;      // tensor-core workspace: A planes | B panel planes | control block
    size_t ws_bytes = 0;
    // fused all-gather target (emm_comm_register_output): every rank's full C
    float *out_local = nullptr;
    int64_t out_ld = 0;
    float *out_peer[8] = {};       // mapped peer buffers (own rank: out_local)
    void *out_opened[8] = {};      // IPC mappings to close
    int *dummy = nullptr;          // completion all-reduce operand
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

struct OutHandle {
    cudaIpcMemHandle_t h;
    int64_t offset;   // bytes from the allocation base to the registered pointer
    int64_t ld;
};

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

int nccl_status(ncclResult_t r) { return r == ncclSuccess ? 0 : EMM_ERR_NCCL_BASE + (int)r; }
int cuda_st(cudaError_t e) { return e == cudaSuccess ? 0 : EMM_ERR_CUDA_BASE + (int)e; }

cudaEvent_t ev_at(Comm *c, size_t i) {
    while (c->evs.size() <= i) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        c->evs.push_back(e);
    }
    return c->evs[i];
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
    if (!n.ok || !comm || !id128 || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) return EMM_ERR_COMM;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    Comm *c = new Comm();
    c->nranks = nranks;
    c->rank = rank;
    cudaGetDevice(&c->dev);
    int st = nccl_status(n.commInitRank(&c->nc, nranks, id, rank));
    if (!st) st = cuda_st(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    if (st) {
        delete c;
        return st;
    }
    *comm = c;
    return 0;
}

extern "C" int emm_comm_unregister_output(void *comm) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    cudaStreamSynchronize(c->comm_stream);
    for (int r = 0; r < 8; ++r) {
        if (c->out_opened[r]) cudaIpcCloseMemHandle(c->out_opened[r]);
        c->out_opened[r] = nullptr;
        c->out_peer[r] = nullptr;
    }
    c->out_local = nullptr;
    c->out_ld = 0;
    return 0;
}

// Collective: every rank registers its M x N (ld_full) full-output buffer;
// CUDA IPC handles are all-gathered over the NCCL communicator and the
// peers' buffers mapped, so emm_sgemm_multi can store C tiles straight into
// them from the GEMM epilogue (NVLink peer stores, no all-gather launch).
extern "C" int emm_comm_register_output(void *comm, float *C_full, int64_t ld_full) {
    if (!comm || !C_full || ld_full < 1) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    Nccl &n = nccl();
    if (!n.ok) return EMM_ERR_COMM;
    emm_comm_unregister_output(comm);
    auto rf = range_fn();
    CUdeviceptr base = 0;
    size_t size = 0;
    if (!rf || rf(&base, &size, reinterpret_cast<CUdeviceptr>(C_full)) != CUDA_SUCCESS) return EMM_ERR_COMM;
    OutHandle mine{};
    int st = cuda_st(cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void *>(base)));
    if (st) return st;
    mine.offset = (int64_t)(reinterpret_cast<CUdeviceptr>(C_full) - base);
    mine.ld = ld_full;
    OutHandle *dev = nullptr;
    if ((st = cuda_st(cudaMalloc(&dev, sizeof(OutHandle) * (c->nranks + 1))))) return st;
    std::vector<OutHandle> all(c->nranks);
    st = cuda_st(cudaMemcpy(dev + c->nranks, &mine, sizeof mine, cudaMemcpyHostToDevice));
    if (!st)
        st = nccl_status(n.allGather(dev + c->nranks, dev, sizeof(OutHandle), ncclUint8, c->nc, c->comm_stream));
    if (!st) st = cuda_st(cudaStreamSynchronize(c->comm_stream));
    if (!st) st = cuda_st(cudaMemcpy(all.data(), dev, sizeof(OutHandle) * c->nranks, cudaMemcpyDeviceToHost));
    cudaFree(dev);
    if (st) return st;
    for (int r = 0; r < c->nranks && !st; ++r) {
        if (all[r].ld != ld_full) st = EMM_ERR_COMM;   // identical layouts required
        if (r == c->rank) {
            c->out_peer[r] = C_full;
            continue;
        }
        void *p = nullptr;
        if (!st) st = cuda_st(cudaIpcOpenMemHandle(&p, all[r].h, cudaIpcMemLazyEnablePeerAccess));
        if (!st) {
            c->out_opened[r] = p;
            c->out_peer[r] = reinterpret_cast<float *>(static_cast<uint8_t *>(p) + all[r].offset);
        }
    }
    if (!st && !c->dummy) st = cuda_st(cudaMalloc(&c->dummy, sizeof(int)));
    if (st) {
        emm_comm_unregister_output(comm);
        return st;
    }
    c->out_local = C_full;
    c->out_ld = ld_full;
    return 0;
}

extern "C" int emm_comm_destroy(void *comm) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    emm_comm_unregister_output(comm);
    if (c->dummy) cudaFree(c->dummy);
    cudaStreamSynchronize(c->comm_stream);
    for (auto e : c->evs) cudaEventDestroy(e);
    if (c->stage) cudaFree(c->stage);
    if (c->ws) cudaFree(c->ws);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    int st = 0;
    if (c->nc) st = nccl_status(nccl().commDestroy(c->nc));
    delete c;
    return st;
}

extern "C" int emm_sgemm_multi(void *comm, char transA, char transB, int64_t M, int64_t N, int64_t K, float alpha,
                               const float *A_local, int64_t lda, float *B, int64_t ldb, int root, float beta,
                               float *C_local, int64_t ldc, float *C_full, int64_t ldc_full, void *stream,
                               emm_math_t math) {
    if (!comm) return EMM_ERR_COMM;
    Comm *c = static_cast<Comm *>(comm);
    Nccl &n = nccl();
    if (!n.ok) return EMM_ERR_COMM;
    if (root < 0 || root >= c->nranks) return EMM_ERR_COMM;
    const bool bN = (transB == 'N' || transB == 'n');
    if (K >= 0 && ldb != (bN ? (K > 1 ? K : 1) : (N > 1 ? N : 1))) return -10;  // panels must be contiguous
    ncclResult_t async_err = ncclSuccess;
    n.getAsyncError(c->nc, &async_err);
    if (async_err != ncclSuccess) return nccl_status(async_err);

    int64_t row0 = 0, rows = 0;
    emm_row_partition(M, c->nranks, c->rank, &row0, &rows);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t b_elems = bN ? K * N : N * K;

    // Gate the communication stream on the caller's stream (B / C ready).
    cudaEvent_t e0 = ev_at(c, 0);
    if (!e0) return EMM_ERR_NOMEM;
    int st = cuda_st(cudaEventRecord(e0, s));
    if (!st) st = cuda_st(cudaStreamWaitEvent(c->comm_stream, e0, 0));
    if (st) return st;

    if ((st = check_args(transA, transB, rows, N, K, lda, ldb, ldc > 0 ? ldc : 1))) return st;
    if ((st = check_device())) return st;
    const int64_t panel = bN ? emm_multi_panel_cols(N) : N;
    // Tensor-core modes: op(A)'s rows are re-buffered ONCE per call into
    // K-major planes in the communicator's cached workspace; each B panel is
    // re-buffered after its broadcast and multiplied (one GEMM launch per
    // panel).  FFMA / alpha == 0 / K == 0 / skinny: one emm_sgemm_ex per panel.
    const bool tc = math != EMM_MATH_FFMA && !(alpha == 0.0f || K == 0) && rows > SKINNY_MAX &&
                    N > SKINNY_MAX && 2.0 * rows * (double)N * K > (double)(1 << 24);
    const int terms = math == EMM_MATH_3XTF32 ? 3 : math == EMM_MATH_TF32_BF16 ? 2 : 1;
    const int planes = terms >= 2 ? 2 : 1;
    const int pmode = math == EMM_MATH_3XTF32 ? PK_FULL3_ : math == EMM_MATH_TF32_BF16 ? PK_FULLX_ : PK_FULL1_;
    const int64_t Kp = tc_kpad(K);
    float *Ap = nullptr, *Bp = nullptr;
    unsigned int *ctrl = nullptr;
    if (tc && rows > 0 && N > 0) {
        const size_t a_bytes = align_up((size_t)planes * rows * Kp * 4, 1024);
        const size_t b_bytes = align_up((size_t)planes * panel * Kp * 4, 1024);
        // stream-ordered reuse: the previous call's kernels on `s` are ordered before this one
        if ((st = grow(&c->ws, &c->ws_bytes, a_bytes + b_bytes + 1024))) return st;
        Ap = reinterpret_cast<float *>(c->ws);
        Bp = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(c->ws) + a_bytes);
        ctrl = reinterpret_cast<unsigned int *>(reinterpret_cast<uint8_t *>(c->ws) + a_bytes + b_bytes);
        PackArgs pa;
        pa.X = A_local; pa.ld = lda; pa.R = rows; pa.kcontig = !(transA == 'N' || transA == 'n');
        pa.out0 = Ap; pa.ld0 = Kp; pa.out1 = Ap + (size_t)rows * Kp; pa.ld1 = Kp; pa.b_side = false;
        st = cuda_st(launch_pack(pmode, pa, nullptr, K, nullptr, s));
    }
    // fused all-gather: C_full was registered -> the GEMM epilogue stores into
    // every rank's C_full directly (tensor-core modes)
    const bool fused = tc && C_full && C_full == c->out_local && ldc_full == c->out_ld;
    auto panel_gemm = [&](const float *bp, int64_t nc, float *cp) -> int {
        if (rows == 0 || nc == 0) return 0;
        if (!tc)
            return emm_sgemm_ex(transA, transB, rows, nc, K, alpha, A_local, lda, bp, ldb, beta, cp, ldc, s, math,
                                nullptr, 0);
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
        PeerOut pe;
        if (fused) {
            pe.n = c->nranks;
            for (int r = 0; r < c->nranks; ++r) pe.base[r] = c->out_peer[r];
            pe.ld = ldc_full;
            pe.row_off = row0;
            pe.col_off = (cp - C_local) / ldc;   // the panel's first column
        }
        if (e == cudaSuccess)
            e = launch_tc_sgemm(terms, ops, rows, nc, K, alpha, beta, cp, ldc, ctrl, 1, nullptr, s,
                                fused ? &pe : nullptr);
        return cuda_st(e);
    };

    if (!st && bN && N > 0) {
        // column panels of B: contiguous K x nc ranges (emm_multi_panel_cols);
        // the GEMM of panel c waits only for panel c's broadcast.
        size_t idx = 1;
        for (int64_t c0 = 0; c0 < N && !st; c0 += panel, ++idx) {
            const int64_t nc = (N - c0 < panel) ? N - c0 : panel;
            float *bp = B + c0 * ldb;
            if (K > 0) st = nccl_status(n.broadcast(bp, bp, (size_t)(K * nc), ncclFloat32, root, c->nc, c->comm_stream));
            cudaEvent_t ev = ev_at(c, idx);
            if (!st && !ev) st = EMM_ERR_NOMEM;
            if (!st) st = cuda_st(cudaEventRecord(ev, c->comm_stream));
            if (!st) st = cuda_st(cudaStreamWaitEvent(s, ev, 0));
            if (!st) st = panel_gemm(bp, nc, C_local + c0 * ldc);
        }
    } else if (!st && N > 0) {
        // transB = 'T': B's stored columns run along K; broadcast it whole
        // (no panel overlap), then one GEMM.
        if (b_elems > 0) st = nccl_status(n.broadcast(B, B, (size_t)b_elems, ncclFloat32, root, c->nc, c->comm_stream));
        cudaEvent_t ev = ev_at(c, 1);
        if (!st) st = cuda_st(cudaEventRecord(ev, c->comm_stream));
        if (!st) st = cuda_st(cudaStreamWaitEvent(s, ev, 0));
        if (!st) st = panel_gemm(B, N, C_local);
    }
    if (st) return st;

    if (C_full && fused) {
        // every rank's epilogue stored its rows into all C_full buffers; a
        // stream-ordered all-reduce completes only after every rank's GEMMs
        // (and their peer stores, fenced at system scope) have finished.
        st = nccl_status(n.allReduce(c->dummy, c->dummy, 1, ncclInt32, ncclSum, c->nc, s));
        if (st) return st;
    } else if (C_full) {
        // all-gather of the row blocks: compact own block into the rank-major
        // staging buffer, P broadcasts in one NCCL group, then unpack (KN6).
        if (ldc_full < (M > 1 ? M : 1)) return -17;
        const size_t need = (size_t)M * (size_t)N * 4;
        if (c->stage_bytes < need) {
            if (c->stage) cudaFree(c->stage);
            c->stage = nullptr;
            c->stage_bytes = 0;
            if ((st = cuda_st(cudaMalloc(&c->stage, need)))) return st;
            c->stage_bytes = need;
        }
        std::vector<int64_t> r0s(c->nranks), rws(c->nranks), offs(c->nranks);
        int64_t off = 0;
        for (int r = 0; r < c->nranks; ++r) {
            emm_row_partition(M, c->nranks, r, &r0s[r], &rws[r]);
            offs[r] = off;
            off += rws[r] * N;
        }
        if (rows > 0 && N > 0)
            st = cuda_st(cudaMemcpy2DAsync(c->stage + offs[c->rank], (size_t)rows * 4, C_local, (size_t)ldc * 4,
                                           (size_t)rows * 4, (size_t)N, cudaMemcpyDeviceToDevice, s));
        if (st) return st;
        {
            n.groupStart();
            for (int r = 0; r < c->nranks; ++r)
                if (rws[r] > 0)
                    n.broadcast(c->stage + offs[r], c->stage + offs[r], (size_t)(rws[r] * N), ncclFloat32, r, c->nc,
                                s);
            st = nccl_status(n.groupEnd());
            if (st) return st;
        }
        st = cuda_st(launch_unpack_rows(c->stage, c->nranks, r0s.data(), rws.data(), N, C_full, ldc_full, s));
        if (st) return st;
    }
    return 0;
}
