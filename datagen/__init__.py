"""Seeded, counter-based synthetic inputs shared by the oracle tests, the GPU
parity tests and ``bench.py``.

This module holds NO arithmetic of the method (no multiply-accumulate, no
tf32 split, no alpha/beta): it only turns (seed, tag, element index) into
float32 values, so that the oracle side and the CUDA side can be fed the very
same bytes, or can regenerate any element independently (SURVEY.md §8(d),
"Data generation").

Generator:

    key(tag, idx, lane) = (seed << 60) ^ (tag << 56) ^ (idx << 1) ^ lane
    h                   = splitmix64(key)
    idx                 = col * stored_rows + row          (column-major)

Distributions (all exactly reproducible on CPU and CUDA, because every step
before the final cast is integer arithmetic, except Box-Muller which is always
evaluated on the CPU in float64):

* ``uniform``   : (h >> 40) * 2^-23 - 1   -> multiples of 2^-23 in [-1, 1)
* ``uniform01`` : (h >> 40) * 2^-24       -> [0, 1)  (same-sign diagnostic)
* ``normal``    : sigma * sqrt(-2 ln u0) cos(2 pi u1), u_l = ((h_l >> 40) + .5) 2^-24
* ``ints``      : ((h >> 40) * 17) >> 24  - 8  -> integers in [-8, 8]
* ``ones`` / ``zeros``

Padding elements (rows .. ld-1 of every column) are NaN so that any read of
padding shows up in a result.

The paper measures on random square matrices (§Results);
there is no dataset, so these synthetic inputs are the workload itself.
"""
from __future__ import annotations

import math

import torch

__all__ = ["splitmix64", "hash_bits", "matrix", "TAG_A", "TAG_B", "TAG_C", "TAG_X"]

TAG_A, TAG_B, TAG_C, TAG_X = 1, 2, 3, 4

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLD = _s64(0x9E3779B97F4A7C15)
_MUL1 = _s64(0xBF58476D1CE4E5B9)
_MUL2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    """logical shift right of int64 bit patterns"""
    return torch.bitwise_and(torch.bitwise_right_shift(z, s), (1 << (64 - s)) - 1)


def splitmix64(key: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors holding uint64 bit patterns
    (wrapping two's-complement multiply)."""
    z = key + _GOLD
    z = torch.bitwise_xor(z, _lsr(z, 30)) * _MUL1
    z = torch.bitwise_xor(z, _lsr(z, 27)) * _MUL2
    return torch.bitwise_xor(z, _lsr(z, 31))


def splitmix64_py(key: int) -> int:
    """Pure-Python twin used to pin the tensor version."""
    z = (key + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def hash_bits(idx: torch.Tensor, tag: int, seed: int = 0, lane: int = 0) -> torch.Tensor:
    """24 random bits (h >> 40) per element index, as int64 in [0, 2^24)."""
    key = torch.bitwise_xor(idx << 1, _s64((seed << 60) ^ (tag << 56) ^ lane))
    return _lsr(splitmix64(key), 40)


def _values(kind: str, idx: torch.Tensor, tag: int, seed: int, sigma: float) -> torch.Tensor:
    if kind == "uniform":
        h = hash_bits(idx, tag, seed)
        return (h - (1 << 23)).to(torch.float32) * (2.0 ** -23)   # exact
    if kind == "uniform01":
        return hash_bits(idx, tag, seed).to(torch.float32) * (2.0 ** -24)
    if kind == "ints":
        h = hash_bits(idx, tag, seed)
        return (((h * 17) >> 24) - 8).to(torch.float32)
    if kind == "normal":
        # Box-Muller in float64 on the CPU only (libm differences between
        # devices must not change the inputs).
        i = idx.cpu()
        u0 = (hash_bits(i, tag, seed, 0).to(torch.float64) + 0.5) * (2.0 ** -24)
        u1 = (hash_bits(i, tag, seed, 1).to(torch.float64) + 0.5) * (2.0 ** -24)
        z = torch.sqrt(-2.0 * torch.log(u0)) * torch.cos((2.0 * math.pi) * u1)
        return (z * sigma).to(torch.float32).to(idx.device)
    if kind == "ones":
        return torch.ones(idx.shape, dtype=torch.float32, device=idx.device)
    if kind == "zeros":
        return torch.zeros(idx.shape, dtype=torch.float32, device=idx.device)
    raise ValueError(f"unknown kind {kind!r}")


def matrix(kind: str, tag: int, rows: int, cols: int, ld: int | None = None, *,
           seed: int = 0, sigma: float = 1.0, device="cpu", pad_value: float = float("nan"),
           chunk_elems: int = 1 << 26) -> torch.Tensor:
    """A column-major float32 matrix: a (rows, cols) tensor with strides
    (1, ld) over a storage of ld*cols floats (padding = ``pad_value``).

    Element (r, c) = value(idx = c*rows + r); independent of ``ld`` and of the
    device it is generated on (``normal`` is always computed on the CPU)."""
    ld = max(1, rows) if ld is None else ld
    if ld < max(1, rows):
        raise ValueError("ld < rows")
    dev = torch.device(device)
    buf = torch.full((max(cols, 0), ld), pad_value, dtype=torch.float32, device=dev)
    if rows > 0 and cols > 0:
        cchunk = max(1, chunk_elems // rows)
        gen_dev = torch.device("cpu") if kind == "normal" else dev
        r = torch.arange(rows, dtype=torch.int64, device=gen_dev)
        for c0 in range(0, cols, cchunk):
            c1 = min(cols, c0 + cchunk)
            c = torch.arange(c0, c1, dtype=torch.int64, device=gen_dev)
            idx = c[:, None] * rows + r[None, :]
            buf[c0:c1, :rows] = _values(kind, idx, tag, seed, sigma).to(dev)
    # (cols, ld) row-major storage == (ld, cols) column-major; keep rows.
    return buf.t()[:rows, :] if rows > 0 else buf.t()[:0, :]


def storage_of(x: torch.Tensor) -> torch.Tensor:
    """The full ld*cols storage (padding included) behind a matrix() view."""
    ld = x.stride(1)          # matrix() views keep stride (1, ld) even for one column
    return torch.as_strided(x, (x.shape[1] * ld,), (1,), x.storage_offset())


def submatrix(kind: str, tag: int, rows: int, cols: int, row_idx, col_idx=None, *, seed: int = 0,
              sigma: float = 1.0, device="cpu") -> torch.Tensor:
    """Selected rows (and columns) of the rows x cols matrix ``matrix(kind,
    tag, rows, cols)`` would give, as a compact column-major (len(row_idx),
    len(col_idx)) tensor — same values element for element, without
    generating the rest (for sampled oracle checks and row-sharded ranks)."""
    dev = torch.device(device)
    gen_dev = torch.device("cpu") if kind == "normal" else dev
    r = torch.as_tensor(row_idx, dtype=torch.int64, device=gen_dev).reshape(-1)
    c = (torch.arange(cols, dtype=torch.int64, device=gen_dev) if col_idx is None
         else torch.as_tensor(col_idx, dtype=torch.int64, device=gen_dev).reshape(-1))
    out = torch.empty((c.numel(), r.numel()), dtype=torch.float32, device=dev)
    cchunk = max(1, (1 << 26) // max(1, r.numel()))
    for c0 in range(0, c.numel(), cchunk):
        cc = c[c0:c0 + cchunk]
        idx = cc[:, None] * rows + r[None, :]
        out[c0:c0 + cc.numel()] = _values(kind, idx, tag, seed, sigma).to(dev)
    return out.t()
