"""Single-kernel entry points over torch CUDA tensors (thin C-ABI wrappers).

Torch supplies device memory and the current stream; the math runs in the
sm_100a kernels of libdroidspeak.so.  Used by the parity tests and by
``bench.py``'s per-kernel roofline measurements.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L

PAGE = 64


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def gemm(a: torch.Tensor, b: torch.Tensor, mode: int = L.EPI_STORE_BF16, resid: torch.Tensor | None = None,
         out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """epilogue(a[M,K] @ b[N,K]^T) on the tcgen05 kernel."""
    assert a.is_cuda and a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.stride(1) == 1 and b.stride(1) == 1
    M, K = a.shape
    N = b.shape[0]
    if out is None:
        dt = torch.float32 if mode in (L.EPI_RESID_F32, L.EPI_STORE_F32) else torch.bfloat16
        out = torch.empty(M, N, device=a.device, dtype=dt)
    with torch.cuda.device(a.device):
        rc = L.lib().ds_gemm(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), out.data_ptr(), out.stride(0),
                             _ptr(resid), resid.stride(0) if resid is not None else 0, M, N, K, mode, _stream(stream))
    L.check(rc)
    return out


def rmsnorm(x: torch.Tensor, gain: torch.Tensor, gather: torch.Tensor | None = None, copy_f32: torch.Tensor | None = None,
            copy_bf16: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    d = x.shape[-1]
    M = gather.numel() if gather is not None else x.numel() // d
    out = torch.empty(M, d, device=x.device, dtype=torch.bfloat16)
    with torch.cuda.device(x.device):
        rc = L.lib().ds_rmsnorm(x.data_ptr(), int(x.dtype == torch.bfloat16), _ptr(gather), M, d, gain.data_ptr(),
                                out.data_ptr(), _ptr(copy_f32), _ptr(copy_bf16), _stream(stream))
    L.check(rc)
    return out


def kv_desc(k: torch.Tensor, v: torch.Tensor, layer_stride: int, head_stride: int, page_stride: int,
            table: torch.Tensor | None, n_layers: int, positions: int) -> L.KvCache:
    return L.KvCache(k.data_ptr(), v.data_ptr(), layer_stride, head_stride, page_stride, _ptr(table), n_layers,
                     positions)


def dense_kv_desc(k: torch.Tensor, v: torch.Tensor) -> L.KvCache:
    """[L, KVH, n, D] dense layout (the reference LayerKV / producer export)."""
    Ln, G, n, D = k.shape
    return kv_desc(k, v, G * n * D, n * D, PAGE * D, None, Ln, n)


def paged_kv_desc(k: torch.Tensor, v: torch.Tensor, table: torch.Tensor, positions: int) -> L.KvCache:
    """[L, pages, KVH, 64, D] paged layout with an int32 block table."""
    Ln, pages, G, ps, D = k.shape
    assert ps == PAGE
    return kv_desc(k, v, pages * G * PAGE * D, PAGE * D, G * PAGE * D, table, Ln, positions)


def attention_prefill(q: torch.Tensor, kv: L.KvCache, layer: int, n_heads: int, n_kv_heads: int, head_dim: int,
                      q_pos0: int = 0, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    n_q = q.shape[0]
    if out is None:
        out = torch.empty(n_q, n_heads * head_dim, device=q.device, dtype=torch.bfloat16)
    with torch.cuda.device(q.device):
        rc = L.lib().ds_attention_prefill(q.data_ptr(), q.stride(0), C.byref(kv), layer, n_q, q_pos0, n_heads,
                                          n_kv_heads, head_dim, out.data_ptr(), out.stride(0), _stream(stream))
    L.check(rc)
    return out


def kv_ingest(src: L.KvCache, dst: L.KvCache, reused: list[int], window: int, n_kv_heads: int, head_dim: int,
              stream=None) -> None:
    arr = (C.c_int32 * max(1, len(reused)))(*reused)
    miss = C.c_int32(-1)
    dev = stream.device if stream is not None else torch.cuda.current_device()
    with torch.cuda.device(dev):
        rc = L.lib().ds_kv_ingest(C.byref(src), C.byref(dst), arr, len(reused), window, n_kv_heads, head_dim,
                                  _stream(stream), C.byref(miss))
    L.check(rc, miss.value, 1)
