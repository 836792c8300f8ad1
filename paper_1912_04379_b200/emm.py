"""ctypes binding of libemm.so (include/emm.h).  Same names as the C ABI,
argument marshalling only.

Matrices are torch float32 tensors laid out COLUMN-major: a (rows, cols)
tensor with strides (1, ld) (e.g. ``x.t().contiguous().t()`` or the views
``datagen.matrix`` returns); ``ld`` is read from ``stride(1)``.  The current
torch CUDA stream is used unless ``stream`` is given.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EMM_LIB: alternative in-tree build of the same library (e.g. the debug
# timeline build libemm_tl.so, tools/timeline.py)
_LIB_PATH = os.path.join(_HERE, os.environ.get("EMM_LIB", "libemm.so"))

MATH = {"3xtf32": 0, "ffma": 1, "1xtf32": 2, "tf32bf16": 3}


class EmmError(RuntimeError):
    def __init__(self, status: int, where: str = "emm"):
        self.status = status
        super().__init__(f"{where}: {strerror(status)} (status {status})")


_lib = None


def lib() -> ctypes.CDLL:
    """Load libemm.so (fails loudly if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python -m paper_1912_04379_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(_LIB_PATH)
    i64, f32, vp, ch, i32, sz = (ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_char,
                                 ctypes.c_int, ctypes.c_size_t)
    gemm13 = [ch, ch, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64]
    L.emm_sgemm.argtypes = gemm13 + [vp]
    L.emm_sgemm.restype = i32
    L.emm_sgemm_ex.argtypes = gemm13 + [vp, i32, vp, sz]
    L.emm_sgemm_ex.restype = i32
    L.emm_sgemm_workspace_bytes.argtypes = [ch, ch, i64, i64, i64, i32]
    L.emm_sgemm_workspace_bytes.restype = sz
    L.emm_sgemm_host.argtypes = gemm13 + [i32]
    L.emm_sgemm_host.restype = i32
    L.emm_release_cache.argtypes = []
    L.emm_release_cache.restype = None
    L.emm_row_partition.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.emm_row_partition.restype = None
    L.emm_multi_panel_cols.argtypes = [i64]
    L.emm_multi_panel_cols.restype = i64
    L.emm_get_unique_id.argtypes = [vp]
    L.emm_get_unique_id.restype = i32
    L.emm_comm_create.argtypes = [ctypes.POINTER(vp), vp, i32, i32]
    L.emm_comm_create.restype = i32
    L.emm_comm_destroy.argtypes = [vp]
    L.emm_comm_destroy.restype = i32
    L.emm_sgemm_multi.argtypes = [vp, ch, ch, i64, i64, i64, f32, vp, i64, vp, i64, i32, f32, vp, i64, vp, i64,
                                  vp, i32]
    L.emm_sgemm_multi.restype = i32
    L.emm_comm_register_output.argtypes = [vp, vp, i64]
    L.emm_comm_register_output.restype = i32
    L.emm_comm_unregister_output.argtypes = [vp]
    L.emm_comm_unregister_output.restype = i32
    L.emm_comm_register_input.argtypes = [vp, vp, sz]
    L.emm_comm_register_input.restype = i32
    L.emm_comm_unregister_input.argtypes = [vp]
    L.emm_comm_unregister_input.restype = i32
    L.emm_debug_comm_create_local.argtypes = [i32, ctypes.POINTER(vp)]
    L.emm_debug_comm_create_local.restype = i32
    L.emm_strerror.argtypes = [i32]
    L.emm_strerror.restype = ctypes.c_char_p
    L.emm_version.argtypes = []
    L.emm_version.restype = ctypes.c_char_p
    L.emm_launch_count.argtypes = []
    L.emm_launch_count.restype = ctypes.c_uint64
    L.emm_profile_enable.argtypes = [i32]
    L.emm_profile_enable.restype = None
    L.emm_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64),
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
    L.emm_profile_read.restype = i32
    _lib = L
    return L


def strerror(status: int) -> str:
    return lib().emm_strerror(int(status)).decode()


def version() -> str:
    return lib().emm_version().decode()


def launch_count() -> int:
    return int(lib().emm_launch_count())


def profile_enable(on: bool = True) -> None:
    lib().emm_profile_enable(1 if on else 0)


def profile_read():
    """(gemm_ms, gemm_launches, other_ms, other_launches) since the last read."""
    g, o = ctypes.c_double(), ctypes.c_double()
    gn, on = ctypes.c_uint64(), ctypes.c_uint64()
    st = lib().emm_profile_read(ctypes.byref(g), ctypes.byref(gn), ctypes.byref(o), ctypes.byref(on))
    if st:
        raise EmmError(st, "emm_profile_read")
    return g.value, gn.value, o.value, on.value


def release_cache() -> None:
    lib().emm_release_cache()


def row_partition(M: int, nranks: int, rank: int):
    r0, n = ctypes.c_int64(), ctypes.c_int64()
    lib().emm_row_partition(M, nranks, rank, ctypes.byref(r0), ctypes.byref(n))
    return r0.value, n.value


def multi_panel_cols(N: int) -> int:
    return int(lib().emm_multi_panel_cols(N))


def get_unique_id() -> bytes:
    """128-byte NCCL unique id (raises EmmError if NCCL cannot be loaded)."""
    idbuf = (ctypes.c_uint8 * 128)()
    st = lib().emm_get_unique_id(ctypes.cast(idbuf, ctypes.c_void_p))
    if st:
        raise EmmError(st, "emm_get_unique_id")
    return bytes(idbuf)


def workspace_bytes(transA, transB, M, N, K, math="3xtf32") -> int:
    return int(lib().emm_sgemm_workspace_bytes(transA.encode(), transB.encode(), M, N, K, MATH[math]))


def _b(c: str) -> bytes:
    return c.encode() if isinstance(c, str) else c


def sgemm_ptr(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, stream=None,
              math="3xtf32", workspace=None, workspace_bytes=0) -> int:
    """Raw C-ABI call with integer device pointers; returns the status code."""
    return lib().emm_sgemm_ex(_b(transA), _b(transB), M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                              stream, MATH[math], workspace, workspace_bytes)


def _ld(x) -> int:
    if x.dim() != 2:
        raise ValueError("expected a 2-D column-major tensor")
    if x.shape[0] > 1 and x.stride(0) != 1:
        raise ValueError("tensor is not column-major (stride(0) must be 1)")
    return max(1, x.stride(1) if x.shape[1] > 1 else max(x.shape[0], 1), x.shape[0])


def _stream_ptr(stream, dev):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    return ctypes.c_void_p(stream.cuda_stream)


def sgemm_ex(A, B, C, alpha=1.0, beta=0.0, transA="N", transB="N", math="3xtf32",
             workspace=None, stream=None) -> None:
    """C <- alpha*op(A)*op(B) + beta*C on torch column-major float32 CUDA tensors.
    A is (M,K) for 'N' / (K,M) for 'T'; B is (K,N) / (N,K); C is (M,N)."""
    import torch
    for t in (A, B, C):
        if t.dtype != torch.float32 or t.device.type != "cuda":
            raise TypeError("A, B, C must be float32 CUDA tensors")
    M, N = C.shape
    K = A.shape[1] if transA in "Nn" else A.shape[0]
    lda, ldb, ldc = _ld(A), _ld(B), _ld(C)
    ws_ptr, ws_n = None, 0
    if workspace is not None:
        ws_ptr, ws_n = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    st = lib().emm_sgemm_ex(_b(transA), _b(transB), M, N, K, float(alpha), A.data_ptr(), lda,
                            B.data_ptr(), ldb, float(beta), C.data_ptr(), ldc,
                            _stream_ptr(stream, C.device), MATH[math], ws_ptr, ws_n)
    if st:
        raise EmmError(st, "emm_sgemm_ex")


def sgemm(A, B, C, alpha=1.0, beta=0.0, transA="N", transB="N", math="3xtf32", stream=None) -> None:
    sgemm_ex(A, B, C, alpha, beta, transA, transB, math, None, stream)


def sgemm_host(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, math="3xtf32") -> None:
    """End-to-end call on HOST buffers (torch CPU tensors / numpy arrays,
    flat column-major storages; pinned memory recommended)."""
    def ptr(x):
        if x is None:
            return None
        if hasattr(x, "data_ptr"):
            return x.data_ptr()
        return x.ctypes.data
    st = lib().emm_sgemm_host(_b(transA), _b(transB), M, N, K, float(alpha), ptr(A), lda, ptr(B), ldb,
                              float(beta), ptr(C), ldc, MATH[math])
    if st:
        raise EmmError(st, "emm_sgemm_host")


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the NCCL id; every rank of the torch.distributed group
    receives the same 128 bytes (the bootstrap of emm_comm_create)."""
    import torch
    import torch.distributed as dist
    raw = get_unique_id() if rank == 0 else bytes(128)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(raw), dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().tolist())


class Comm:
    """NCCL communicator for emm_sgemm_multi, bootstrapped over an existing
    torch.distributed process group (the 128-byte id is broadcast with it)."""

    def __init__(self, rank: int, nranks: int, group=None):
        import torch
        import torch.distributed as dist
        raw = broadcast_unique_id(rank, group)
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(raw)
        h = ctypes.c_void_p()
        st = lib().emm_comm_create(ctypes.byref(h), ctypes.cast(idbuf, ctypes.c_void_p), nranks, rank)
        if st:
            raise EmmError(st, "emm_comm_create")
        self.handle, self.rank, self.nranks = h, rank, nranks

    def register_output(self, C_full) -> None:
        """Collective: map every rank's C_full so emm_sgemm_multi fuses the
        all-gather into the GEMM epilogue (peer stores over NVLink)."""
        st = lib().emm_comm_register_output(self.handle, C_full.data_ptr(), _ld(C_full))
        if st:
            raise EmmError(st, "emm_comm_register_output")

    def unregister_output(self) -> None:
        lib().emm_comm_unregister_output(self.handle)

    def register_input(self, B) -> None:
        """Collective: register this rank's B buffer (source on root, receive
        buffer elsewhere) so emm_sgemm_multi forwards B by peer copies along
        the ring (copy engines + flags) instead of ncclBroadcast."""
        nbytes = ((B.shape[1] - 1) * _ld(B) + B.shape[0]) * 4 if B.numel() else 0
        st = lib().emm_comm_register_input(self.handle, B.data_ptr(), nbytes)
        if st:
            raise EmmError(st, "emm_comm_register_input")

    def unregister_input(self) -> None:
        lib().emm_comm_unregister_input(self.handle)

    def close(self):
        if self.handle:
            lib().emm_comm_destroy(self.handle)
            self.handle = None


class _LocalComm(Comm):
    def __init__(self, handle, rank, nranks):  # noqa: D401 - built by local_comms()
        self.handle, self.rank, self.nranks = handle, rank, nranks


def local_comms(nranks: int):
    """emm_debug_comm_create_local: `nranks` virtual ranks on the current
    device (test harness for the P > 1 paths on one GPU); returns one Comm per
    rank.  Each rank needs its own stream; B (and a gathered C_full) must be
    registered."""
    arr = (ctypes.c_void_p * nranks)()
    st = lib().emm_debug_comm_create_local(nranks, arr)
    if st:
        raise EmmError(st, "emm_debug_comm_create_local")
    return [_LocalComm(ctypes.c_void_p(arr[r]), r, nranks) for r in range(nranks)]


def sgemm_multi(comm: Comm, M, N, K, A_local, B, C_local, alpha=1.0, beta=0.0, transA="N", transB="N",
                root=0, C_full=None, math="3xtf32", stream=None) -> None:
    """Row-sharded SGEMM (emm_sgemm_multi): A_local/C_local are this rank's
    row blocks (emm_row_partition), B the full op(B) storage (filled on root)."""
    ldc_full = _ld(C_full) if C_full is not None else 0
    st = lib().emm_sgemm_multi(comm.handle, _b(transA), _b(transB), M, N, K, float(alpha),
                               A_local.data_ptr(), _ld(A_local), B.data_ptr(), _ld(B), root,
                               float(beta), C_local.data_ptr(), _ld(C_local),
                               C_full.data_ptr() if C_full is not None else None, ldc_full,
                               _stream_ptr(stream, C_local.device), MATH[math])
    if st:
        raise EmmError(st, "emm_sgemm_multi")
