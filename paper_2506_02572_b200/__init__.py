"""HATA decode hot path on B200 (sm_100a): thin Python binding over libhata.

Same names as the C ABI (include/hata.h).  This layer only marshals torch
tensors (device memory, streams) into pointers/strides; every step of the
method runs in the CUDA kernels of libhata.so.  There is no fallback path.

Tensor conventions (see include/hata.h):
  K, V   [B, H_kv, cap, d]  bf16|fp32, last dim contiguous
  codes  [B, H_kv, cap, rbits//32] int32 (uint32 bit patterns), rows packed
  W      [H_kv, d, rbits]   same dtype as K
  q      [B, H_q, d]
  n, pos [B] int64 on the device
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import HataError, Strides  # noqa: F401

__all__ = ["set_option", "hash_keys", "prefill_write", "append", "decode_topk_attn", "decode_step", "decode_step_paged", "decode_workspace_size", "decode_ranks",
           "shard_candidates", "shard_select", "shard_partial_attn", "shard_combine", "HataError", "lib"]


def lib():
    return _lib.load()


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.HATA_BF16
    if t.dtype == torch.float32:
        return _lib.HATA_F32
    raise HataError(f"unsupported dtype {t.dtype}")


def _dt_of(dtype: torch.dtype) -> int:
    return _lib.HATA_BF16 if dtype == torch.bfloat16 else _lib.HATA_F32


def _strides4(t: torch.Tensor) -> Strides:
    if t.dim() != 4 or t.stride(3) != 1:
        raise HataError("expected a [B, H, cap, x] tensor with a contiguous last dim")
    return Strides(t.stride(0), t.stride(1), t.stride(2))


def _p(t):
    """Device pointer of ``t``.  Callers pass tensors that stay referenced
    until the call returns: a temporary (e.g. ``x.contiguous()``) freed before
    the asynchronous launch may be handed by the caching allocator to the next
    copy on the stream and overwritten before the kernel reads it."""
    return None if t is None else t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise HataError("all tensors must be CUDA tensors (no CPU path)")


def _need_kv(K, V):
    """K/V caches: CUDA tensors, or -- HATA-off -- pinned host
    tensors, which CUDA maps into the device address space (UVA): the decode
    kernel gathers only the selected rows from host memory itself."""
    for t in (K, V):
        if not (t.is_cuda or (t.device.type == "cpu" and t.is_pinned())):
            raise HataError("K/V must be CUDA tensors or pinned host tensors (HATA-off)")


def set_option(name: str, value: int):
    """hata_set_option: "selection_hint", "pdl" or "cooperative" (process-wide, default on)."""
    opt = {"selection_hint": _lib.HATA_OPT_SELECTION_HINT, "pdl": _lib.HATA_OPT_PDL,
           "cooperative": _lib.HATA_OPT_COOPERATIVE}[name]
    _lib.check(lib().hata_set_option(opt, int(value)), "hata_set_option")


def hash_keys(K, W, codes, t0: int = 0, n: int | None = None, stream=None):
    """Alg. 1 lines 2-5: codes[:, :, t0:t0+n] = HashEncode(K[:, :, t0:t0+n]) (in place)."""
    _need_cuda(K, W, codes)
    W = W.contiguous()
    B, Hkv, cap, d = K.shape
    rbits = W.shape[2]
    n = cap - t0 if n is None else n
    _lib.check(lib().hata_hash_keys(_p(K), _strides4(K), _dt(K), _p(W), B, Hkv, d, rbits, t0, n, cap,
                                    _p(codes), _strides4(codes), _stream(stream)), "hata_hash_keys")
    return codes


def prefill_write(K_src, V_src, W, K, V, codes, t0: int = 0, stream=None):
    """NEXT-1: K/V chunk [B, H_kv, n, d] -> cache rows [t0, t0+n) and their
    codes, keys read once (hata_prefill_write)."""
    _need_cuda(K_src, V_src, W, K, V, codes)
    W = W.contiguous()
    B, Hkv, n, d = K_src.shape
    if K_src.stride() != V_src.stride() or K.stride() != V.stride():
        raise HataError("K and V must share strides (source and cache)")
    _lib.check(lib().hata_prefill_write(_p(K_src), _p(V_src), _strides4(K_src), _p(K), _p(V), _strides4(K), _dt(K),
                                        _p(W), B, Hkv, d, W.shape[2], t0, n, K.shape[2], _p(codes), _strides4(codes),
                                        _stream(stream)), "hata_prefill_write")


def append(k_new, v_new, W, K, V, codes, pos, stream=None):
    """Alg. 3 lines 2-9: write k_new/v_new and HashEncode(k_new) at row pos[b] (in place)."""
    _need_cuda(k_new, v_new, W, codes, pos)
    _need_kv(K, V)
    k_new, v_new = k_new.contiguous(), v_new.contiguous()
    B, Hkv, cap, d = K.shape
    if K.stride() != V.stride():
        raise HataError("K and V must share strides")
    _lib.check(lib().hata_append(_p(k_new), _p(v_new), _dt(K), _p(W), _p(K), _p(V),
                                 _strides4(K), _p(codes), _strides4(codes), _p(pos), cap, B, Hkv, d, W.shape[2],
                                 _stream(stream)), "hata_append")


def decode_workspace_size(B, Hq, Hkv, d, rbits, n_max, k, dtype=torch.bfloat16) -> int:
    return int(lib().hata_decode_workspace_size(B, Hq, Hkv, d, rbits, n_max, k, _dt_of(dtype)))


def decode_ranks(B, Hq, Hkv, d, rbits, n_max, k, dtype=torch.bfloat16) -> int:
    return int(lib().hata_decode_ranks(B, Hq, Hkv, d, rbits, n_max, k, _dt_of(dtype)))


def decode_topk_attn(q, K, V, codes, W, n, k: int, n_max: int | None = None, scale: float = 0.0, out=None,
                     out_dtype=torch.float32, out_idx=None, out_score=None, out_qcodes=None, workspace=None,
                     stream=None):
    """Alg. 3 lines 6, 10-17 over caches already holding the new token.
    Returns ``out`` [B, H_q, d]."""
    _need_cuda(q, codes, W, n)
    _need_kv(K, V)
    q = q.contiguous()
    B, Hq, d = q.shape
    Hkv, rbits = K.shape[1], W.shape[2]
    if n_max is None:
        n_max = K.shape[2]
    if out is None:
        out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    if K.stride() != V.stride():
        raise HataError("K and V must share strides")
    ws = decode_workspace_size(B, Hq, Hkv, d, rbits, n_max, k, K.dtype)
    if ws and (workspace is None or workspace.numel() * workspace.element_size() < ws):
        workspace = torch.zeros(ws, dtype=torch.uint8, device=q.device)
    _lib.check(lib().hata_decode_topk_attn(
        _p(q), _p(K), _p(V), _strides4(K), _dt(K), _p(codes), _strides4(codes), _p(W), B, Hq, Hkv, d,
        rbits, _p(n), n_max, k, scale, _p(out), _dt(out), _p(out_idx), _p(out_score), _p(out_qcodes),
        _p(workspace) if ws else None, ws, _stream(stream)), "hata_decode_topk_attn")
    return out


def decode_step(q, k_new, v_new, K, V, codes, W, n, k: int, n_max: int | None = None, scale: float = 0.0,
                out=None, out_dtype=torch.float32, out_idx=None, out_score=None, out_qcodes=None, workspace=None,
                stream=None):
    """Alg. 3 lines 2-17 in one launch: append k_new/v_new (and the key code) at
    row n[b]-1, then decode.  ``n`` counts the new token.  Returns ``out``."""
    _need_cuda(q, k_new, v_new, codes, W, n)
    _need_kv(K, V)
    q, k_new, v_new = q.contiguous(), k_new.contiguous(), v_new.contiguous()
    B, Hq, d = q.shape
    Hkv, cap, rbits = K.shape[1], K.shape[2], W.shape[2]
    if n_max is None:
        n_max = cap
    if out is None:
        out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    if K.stride() != V.stride():
        raise HataError("K and V must share strides")
    ws = decode_workspace_size(B, Hq, Hkv, d, rbits, n_max, k, K.dtype)
    if ws and (workspace is None or workspace.numel() * workspace.element_size() < ws):
        workspace = torch.zeros(ws, dtype=torch.uint8, device=q.device)
    _lib.check(lib().hata_decode_step(
        _p(q), _p(k_new), _p(v_new), _p(K), _p(V), _strides4(K), _dt(K),
        _p(codes), _strides4(codes), _p(W), B, Hq, Hkv, d, rbits, _p(n), n_max, cap, k, scale, _p(out), _dt(out),
        _p(out_idx), _p(out_score), _p(out_qcodes), _p(workspace) if ws else None, ws, _stream(stream)),
        "hata_decode_step")
    return out


def decode_step_paged(q, k_new, v_new, K, V, codes, W, page_table, n, k: int, n_max: int, scale: float = 0.0,
                      out=None, out_dtype=torch.float32, out_idx=None, out_score=None, out_qcodes=None,
                      workspace=None, stream=None):
    """hata_decode_step over paged pools.  K, V: [pages, H_kv, page_size, d]
    views (any page/head/token strides, d contiguous); codes: [pages, H_kv,
    page_size, rbits//32]; page_table: int32 [B, max_pages] on the device."""
    _need_cuda(q, k_new, v_new, codes, W, page_table, n)
    _need_kv(K, V)
    q, k_new, v_new = q.contiguous(), k_new.contiguous(), v_new.contiguous()
    B, Hq, d = q.shape
    Hkv, page_size, rbits = K.shape[1], K.shape[2], W.shape[2]
    if page_table.dtype != torch.int32 or page_table.dim() != 2 or not page_table.is_contiguous():
        raise HataError("page_table must be a contiguous int32 [B, max_pages] tensor")
    if out is None:
        out = torch.empty(B, Hq, d, dtype=out_dtype, device=q.device)
    if K.stride() != V.stride():
        raise HataError("K and V must share strides")
    ws = decode_workspace_size(B, Hq, Hkv, d, rbits, n_max, k, K.dtype)
    if ws and (workspace is None or workspace.numel() * workspace.element_size() < ws):
        workspace = torch.zeros(ws, dtype=torch.uint8, device=q.device)
    _lib.check(lib().hata_decode_step_paged(
        _p(q), _p(k_new), _p(v_new), _p(K), _p(V), _strides4(K), _dt(K), _p(codes), _strides4(codes),
        _p(page_table), page_table.shape[1], page_size, _p(W), B, Hq, Hkv, d, rbits, _p(n), n_max, k, scale,
        _p(out), _dt(out), _p(out_idx), _p(out_score), _p(out_qcodes), _p(workspace) if ws else None, ws,
        _stream(stream)), "hata_decode_step_paged")
    return out


def shard_candidates(q, codes, W, n_local, n_local_max: int, token_offset: int, k: int, cand_D, cand_idx,
                     workspace=None, stream=None):
    _need_cuda(q, codes, W, n_local, cand_D, cand_idx)
    q = q.contiguous()
    B, Hq, d = q.shape
    Hkv, rbits = codes.shape[1], W.shape[2]
    ws = decode_workspace_size(B, Hq, Hkv, d, rbits, n_local_max, k, q.dtype)
    if ws and (workspace is None or workspace.numel() * workspace.element_size() < ws):
        workspace = torch.zeros(ws, dtype=torch.uint8, device=q.device)
    _lib.check(lib().hata_shard_candidates(
        _p(q), _dt(q), _p(codes), _strides4(codes), _p(W), B, Hq, Hkv, d, rbits, _p(n_local),
        n_local_max, token_offset, k, _p(cand_D), _p(cand_idx), _p(workspace) if ws else None, ws,
        _stream(stream)), "hata_shard_candidates")


def shard_select(all_D, all_idx, n_total, lo: int, hi: int, G: int, rbits: int, own_idx, own_cnt, sel_idx=None,
                 sel_score=None, stream=None):
    """all_D / all_idx: [P, B, H_kv, k] views whose rank blocks may be strided
    (e.g. the two halves of one gathered [P, 2, B, H_kv, k] buffer)."""
    _need_cuda(all_D, all_idx, n_total, own_idx, own_cnt)
    P, B, Hkv, k = all_D.shape
    if all_D.stride()[1:] != (Hkv * k, k, 1) or all_idx.stride() != all_D.stride():
        raise HataError("candidate blocks must be [B, H_kv, k] contiguous with one rank stride")
    _lib.check(lib().hata_shard_select(_p(all_D), _p(all_idx), all_D.stride(0), P, B, Hkv, k, G, rbits,
                                       _p(n_total), lo, hi, _p(own_idx), _p(own_cnt), _p(sel_idx), _p(sel_score),
                                       _stream(stream)), "hata_shard_select")


def shard_partial_attn(q, K, V, own_idx, own_cnt, k: int, partial, scale: float = 0.0, stream=None):
    """partial: [splits, B, H_q, d + 2] fp32 (splits CTAs per (b, KV head))."""
    _need_cuda(q, K, V, own_idx, own_cnt, partial)
    q = q.contiguous()
    B, Hq, d = q.shape
    Hkv = K.shape[1]
    splits = partial.shape[0] if partial.dim() == 4 else 1
    _lib.check(lib().hata_shard_partial_attn(_p(q), _p(K), _p(V), _strides4(K), _dt(K), _p(own_idx),
                                             _p(own_cnt), B, Hq, Hkv, d, k, scale, splits, _p(partial),
                                             _stream(stream)), "hata_shard_partial_attn")


def shard_combine(partials, out, stream=None):
    _need_cuda(partials, out)
    P, B, Hq, d2 = partials.shape
    _lib.check(lib().hata_shard_combine(_p(partials), P, B, Hq, d2 - 2, _p(out), _dt(out), _stream(stream)),
               "hata_shard_combine")
