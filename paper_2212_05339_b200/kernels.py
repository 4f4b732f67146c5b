"""Typed torch-tensor wrappers over the C-ABI (include/elixir_b200.h).

Every function here launches native code from libelixir_b200.so on the
given (or current) CUDA stream; there is no CPU or PyTorch fallback. Inputs
are validated for device/dtype/contiguity before the call; the library
validates sizes and alignment and returns typed errors (_lib.check).
"""

from __future__ import annotations

import ctypes
import json
import os
import threading
from pathlib import Path
from typing import Sequence

import torch

from . import _lib
from .errors import ValidationError

_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16}


def elx_dtype(dt: torch.dtype) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise ValidationError(f"unsupported dtype {dt}") from None


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def event_record(event: torch.cuda.Event, stream=None) -> None:
    """Record `event` on `stream`; inside a CUDA-graph capture as an external
    event-record node that every replay re-records (elx_event_record). The
    event must already exist (torch creates it on its first record)."""
    if not event.cuda_event:
        raise ValidationError("event_record needs an event that was recorded once before (created)")
    _lib.check(_lib.load().elx_event_record(event.cuda_event, _stream(stream)), "elx_event_record")


def _cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ValidationError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValidationError(f"{what} must be contiguous")


def chunk_pack(chunk: torch.Tensor, members: Sequence[tuple[torch.Tensor | None, int]],
               used_len: int | None = None, stream=None) -> None:
    """K1: chunk[off:off+t.numel()] <- t for (t, off) in members; zero the tail
    [used_len, chunk.numel()) when used_len is given. A member with t=None and
    an explicit numel given as (None, off, numel) writes zeros."""
    lib = _lib.load()
    _cuda(chunk, "chunk")
    arr = (_lib.Member * max(1, len(members)))()
    keep = []
    for i, m in enumerate(members):
        if m[0] is None:
            arr[i].ext, arr[i].offset, arr[i].numel, arr[i].ext_dtype = None, int(m[1]), int(m[2]), elx_dtype(chunk.dtype)
            continue
        t = m[0]
        if not t.is_contiguous():
            t = t.contiguous()
        _cuda(t, "member")
        keep.append(t)
        arr[i].ext, arr[i].offset, arr[i].numel, arr[i].ext_dtype = t.data_ptr(), int(m[1]), t.numel(), elx_dtype(t.dtype)
    used = chunk.numel() if used_len is None else int(used_len)
    rc = lib.elx_chunk_pack(chunk.data_ptr(), elx_dtype(chunk.dtype), chunk.numel(), used,
                            ctypes.addressof(arr), len(members), _stream(stream))
    _lib.check(rc, "elx_chunk_pack")


def chunk_unpack(chunk: torch.Tensor, members: Sequence[tuple[torch.Tensor, int]], stream=None) -> None:
    """K1 reverse: t <- chunk[off:off+t.numel()] for (t, off) in members."""
    lib = _lib.load()
    _cuda(chunk, "chunk")
    arr = (_lib.Member * max(1, len(members)))()
    for i, (t, off) in enumerate(members):
        _cuda(t, "member")
        if off + t.numel() > chunk.numel():
            raise ValidationError("member exceeds chunk")
        arr[i].ext, arr[i].offset, arr[i].numel, arr[i].ext_dtype = t.data_ptr(), int(off), t.numel(), elx_dtype(t.dtype)
    rc = lib.elx_chunk_unpack(chunk.data_ptr(), elx_dtype(chunk.dtype), ctypes.addressof(arr),
                              len(members), _stream(stream))
    _lib.check(rc, "elx_chunk_unpack")


def _ptr_array(ptrs: Sequence[int]):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def fetch(block: torch.Tensor, shard_ptrs: Sequence[int], shard_len: int, stream=None, engine: str = "sm",
          rank: int = 0) -> None:
    """K2: block[r*S:(r+1)*S] <- shard r (device pointers, local or peer-mapped).
    engine "sm": the fetch kernel (TMA bulk copies); "ce": the copy engines
    (one cudaMemcpyAsync per rank, spread over up to four streams forked from
    `stream` and joined back), leaving every SM to the compute stream. `rank`
    (the caller's) rotates the order of the peer reads to start at rank+1
    (elx_fetch_ranked), so the ranks of one all-gather do not all read the
    same peer at once."""
    lib = _lib.load()
    _cuda(block, "block")
    if block.numel() < len(shard_ptrs) * shard_len:
        raise ValidationError("block smaller than world * shard_len")
    if engine not in ("sm", "ce"):
        raise ValidationError(f"fetch engine must be 'sm' or 'ce', not {engine!r}")
    arr = _ptr_array(shard_ptrs)
    rc = lib.elx_fetch_ranked(block.data_ptr(), ctypes.addressof(arr), int(shard_len), int(rank), len(shard_ptrs),
                              elx_dtype(block.dtype), 0 if engine == "sm" else 1, _stream(stream))
    _lib.check(rc, "elx_fetch" if engine == "sm" else "elx_fetch_ce")


def enable_peer_access(peer_device: int) -> None:
    """Let kernels on the current device read/write memory on `peer_device`
    (NVLink P2P; a no-op when already enabled or when it is this device)."""
    _lib.check(_lib.load().elx_enable_peer_access(int(peer_device)), "elx_enable_peer_access")


def ipc_open(handle: bytes) -> int:
    """Map a peer process's allocation (64-byte cudaIpcMemHandle_t) into the
    current device's context; returns its base pointer here."""
    if len(handle) != 64:
        raise ValidationError("a CUDA IPC handle is 64 bytes")
    buf = ctypes.create_string_buffer(bytes(handle), 64)
    out = ctypes.c_void_p()
    _lib.check(_lib.load().elx_ipc_open(buf, ctypes.byref(out)), "elx_ipc_open")
    return int(out.value)


def ipc_close(ptr: int) -> None:
    _lib.check(_lib.load().elx_ipc_close(ctypes.c_void_p(ptr)), "elx_ipc_close")


def device_barrier(pad_ptrs: Sequence[int], rank: int, epoch: int, stream=None) -> None:
    """Stream-ordered cross-rank barrier over peer-mapped int32[world] signal
    pads (pad_ptrs[r] = rank r's pad as a pointer usable on this device)."""
    lib = _lib.load()
    arr = _ptr_array(pad_ptrs)
    rc = lib.elx_device_barrier(ctypes.addressof(arr), len(pad_ptrs), int(rank), int(epoch), _stream(stream))
    _lib.check(rc, "elx_device_barrier")


def peer_sum_f64(dst: torch.Tensor, peer_ptrs: Sequence[int], count: int, stream=None) -> None:
    """dst[:count] = sum over ranks (rank order) of peer_ptrs[r][:count] (fp64)."""
    _cuda(dst, "dst")
    if dst.dtype != torch.float64 or dst.numel() < count:
        raise ValidationError("peer_sum_f64 needs a float64 destination of >= count elements")
    arr = _ptr_array(peer_ptrs)
    rc = _lib.load().elx_peer_sum_f64(dst.data_ptr(), ctypes.addressof(arr), int(count), len(peer_ptrs),
                                      _stream(stream))
    _lib.check(rc, "elx_peer_sum_f64")


STEP_SCALARS = _lib.STEP_SCALARS


def new_step_scalars(device) -> torch.Tensor:
    """A zeroed step-scalar block (include/elixir_b200.h, K3): [0] sum of
    squares, [1] overflow flag, [2] completed steps, then the release kernels'
    arrival ticket and per-CTA partial slots (deterministic norm)."""
    return torch.zeros(STEP_SCALARS, dtype=torch.float64, device=device)


def _check_scalars(step_scalars: torch.Tensor) -> None:
    if step_scalars.dtype != torch.float64 or not step_scalars.is_cuda or not step_scalars.is_contiguous():
        raise ValidationError("step_scalars must be a contiguous CUDA float64 tensor")
    if step_scalars.numel() < STEP_SCALARS:
        raise ValidationError(f"step_scalars must hold the {STEP_SCALARS}-double step-scalar block "
                              "(kernels.new_step_scalars)")


def release(grad_shard: torch.Tensor | None, src_ptrs: Sequence[int], n: int, dtype: torch.dtype,
            inv_scale: float, step_scalars: torch.Tensor, stream=None) -> None:
    """K3: grad_shard[:n] = (sum_r src_r[:n] in rank order, fp32) * inv_scale,
    accumulating sum(g^2) into step_scalars[0] (fixed order, deterministic) and
    overflow into step_scalars[1]. grad_shard=None: norm/overflow only (world-1
    in-place chunks)."""
    release_batch([(grad_shard, src_ptrs, n)], dtype, inv_scale, step_scalars, stream=stream)


def release_batch(segs: Sequence[tuple[torch.Tensor | None, Sequence[int], int]], dtype: torch.dtype,
                  inv_scale: float, step_scalars: torch.Tensor, stream=None) -> None:
    """K3 over several segments in ONE launch (per 16 segments): every chunk due
    at one reduce position. segs: (grad_shard or None, per-rank source device
    pointers, valid elements n)."""
    lib = _lib.load()
    _check_scalars(step_scalars)
    if not segs:
        return
    world = len(segs[0][1])
    arr = (_lib.ReleaseSeg * len(segs))()
    for i, (g, ptrs, n) in enumerate(segs):
        if len(ptrs) != world:
            raise ValidationError("every release segment needs one source per rank")
        if g is not None:
            _cuda(g, "grad_shard")
            if g.dtype != torch.float32 or g.numel() < n:
                raise ValidationError("grad_shard must be float32 with >= n elements")
        arr[i].g = None if g is None else g.data_ptr()
        for r, p in enumerate(ptrs):
            arr[i].src[r] = p
        arr[i].n = int(n)
    rc = lib.elx_release_batch(ctypes.addressof(arr), len(segs), world, elx_dtype(dtype), float(inv_scale),
                               step_scalars.data_ptr(), _stream(stream))
    _lib.check(rc, "elx_release_batch")


def release_geometry(lengths: Sequence[int], world: int, dtype: torch.dtype = torch.bfloat16) -> tuple[int, int]:
    """(ctas, tile_vecs) of one K3 launch over segments of these lengths on the
    current device: the fixed summation order of its sum of squares."""
    lib = _lib.load()
    n = (ctypes.c_int64 * max(1, len(lengths)))(*[int(x) for x in lengths])
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.elx_release_geometry(ctypes.addressof(n), len(lengths), int(world), elx_dtype(dtype),
                                        ctypes.byref(a), ctypes.byref(b)), "elx_release_geometry")
    return a.value, b.value


class AdamTable:
    """Device-resident K4 segment table (built once per plan; static pointers)."""

    def __init__(self, segs: Sequence[tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor,
                                            torch.Tensor, int]], device):
        host = (_lib.AdamSeg * max(1, len(segs)))()
        tile = 0
        self.valid_elements = 0
        for i, (p32, m, v, g, p16, n) in enumerate(segs):
            for t in (p32, m, v, g, p16):
                _cuda(t, "adam segment tensor")
            host[i].p32, host[i].m, host[i].v = p32.data_ptr(), m.data_ptr(), v.data_ptr()
            host[i].g, host[i].p16, host[i].n, host[i].tile0 = g.data_ptr(), p16.data_ptr(), int(n), tile
            host[i].g_dtype = elx_dtype(g.dtype)
            tile += -(-int(n) // _lib.ADAM_TILE)
            self.valid_elements += int(n)
        self.nseg = len(segs)
        self.ntiles = tile
        raw = bytes(host)
        self.dev = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)
        self._keep = [s[:5] for s in segs]


def _hp(hp: dict, p16_dtype: torch.dtype, grad_scale: float, bias_tables=None):
    h = _lib.AdamHP(hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"],
                    hp.get("max_norm", 0.0) or 0.0, float(grad_scale), elx_dtype(p16_dtype), 0)
    if bias_tables is not None:
        bc1, bc2s = bias_tables
        h.bc1_table, h.bc2s_table, h.table_len = bc1.data_ptr(), bc2s.data_ptr(), bc1.numel()
    return h


class BiasTables:
    """Device tables of Adam's bias corrections for the device-step mode of
    K4: bc1[t] = 1 - beta1**t (float64), bc2s[t] = float32((1 - beta2**t)**0.5),
    computed on the host with the oracle's float64 formulas."""

    def __init__(self, beta1: float, beta2: float, device, length: int = 4096):
        self.beta1, self.beta2, self.device = beta1, beta2, device
        self.bc1 = self.bc2s = None
        self._build(length)

    def _build(self, length: int) -> None:
        import numpy as np
        t = np.arange(length, dtype=np.float64)
        bc1 = 1.0 - np.power(self.beta1, t)
        bc2s = np.power(1.0 - np.power(self.beta2, t), 0.5).astype(np.float32)
        bc1[0] = 1.0  # t = 0 is never used (steps start at 1); keep it finite
        bc2s[0] = 1.0
        self.bc1 = torch.from_numpy(bc1).to(self.device)
        self.bc2s = torch.from_numpy(bc2s).to(self.device)

    def ensure(self, max_step: int) -> None:
        if max_step + 2 > self.bc1.numel():
            self._build(max(2 * self.bc1.numel(), max_step + 2))

    def pair(self):
        return self.bc1, self.bc2s


def adam(table: AdamTable, hp: dict, step: int, step_scalars: torch.Tensor, p16_dtype: torch.dtype,
         stream=None, grad_scale: float = 1.0, bias_tables: BiasTables | None = None, max_ctas: int = 0) -> None:
    """K4 over every segment of `table` in one launch. Segments whose
    gradient is in the compute dtype are unscaled by `grad_scale` in-register.
    step >= 1: host step; step == 0: device step (step_scalars[2] + 1) with
    `bias_tables`. max_ctas > 0 caps the grid (an update sharing the GPU)."""
    lib = _lib.load()
    h = _hp(hp, p16_dtype, grad_scale, None if bias_tables is None else bias_tables.pair())
    h.max_ctas = int(max_ctas)
    rc = lib.elx_adam(table.dev.data_ptr(), table.nseg, table.ntiles, ctypes.byref(h), int(step),
                      step_scalars.data_ptr(), _stream(stream))
    _lib.check(rc, "elx_adam")


def cpu_adam(segs: Sequence[tuple[torch.Tensor, ...]], hp: dict, step: int, scalars_host: Sequence[float],
             p16_dtype: torch.dtype, threads: int, grad_scale: float = 1.0) -> None:
    """Host AdamW (same bits as K4) over CPU tensors (p32, m, v, g, p16, n)."""
    lib = _lib.load()
    arr = (_lib.CpuSeg * max(1, len(segs)))()
    for i, (p32, m, v, g, p16, n) in enumerate(segs):
        for t in (p32, m, v, g, p16):
            if t.is_cuda or not t.is_contiguous():
                raise ValidationError("cpu_adam needs contiguous host tensors")
        arr[i].p32, arr[i].m, arr[i].v = p32.data_ptr(), m.data_ptr(), v.data_ptr()
        arr[i].g, arr[i].p16, arr[i].n = g.data_ptr(), p16.data_ptr(), int(n)
        arr[i].g_dtype = elx_dtype(g.dtype)
    h = _hp(hp, p16_dtype, grad_scale)
    sc = (ctypes.c_double * 2)(float(scalars_host[0]), float(scalars_host[1]))
    rc = lib.elx_cpu_adam(ctypes.addressof(arr), len(segs), ctypes.byref(h), int(step),
                          ctypes.addressof(sc), int(threads))
    _lib.check(rc, "elx_cpu_adam")


def norm_finalize(step_scalars: torch.Tensor, max_norm: float, out3: torch.Tensor, stream=None) -> None:
    lib = _lib.load()
    rc = lib.elx_norm_finalize(step_scalars.data_ptr(), float(max_norm or 0.0), out3.data_ptr(),
                               _stream(stream))
    _lib.check(rc, "elx_norm_finalize")


def step_reset(step_scalars: torch.Tensor, stream=None) -> None:
    lib = _lib.load()
    _lib.check(lib.elx_step_reset(step_scalars.data_ptr(), _stream(stream)), "elx_step_reset")


def step_advance(step_scalars: torch.Tensor, stream=None) -> None:
    """Device-side end of step: count it unless it overflowed; clear Σg²/flag."""
    lib = _lib.load()
    _lib.check(lib.elx_step_advance(step_scalars.data_ptr(), _stream(stream)), "elx_step_advance")


def copy_h2d(dst: torch.Tensor, src_host: torch.Tensor, nbytes: int | None = None, stream=None,
             event: torch.cuda.Event | None = None) -> None:
    """K6: pinned host -> HBM on `stream` (copy engine)."""
    lib = _lib.load()
    nb = src_host.numel() * src_host.element_size() if nbytes is None else int(nbytes)
    ev = event.cuda_event if event is not None else None
    rc = lib.elx_copy_h2d(dst.data_ptr(), src_host.data_ptr(), nb, _stream(stream), ev)
    _lib.check(rc, "elx_copy_h2d")


def copy_d2h(dst_host: torch.Tensor, src: torch.Tensor, nbytes: int | None = None, stream=None,
             event: torch.cuda.Event | None = None) -> None:
    """K6: HBM -> pinned host on `stream` (copy engine)."""
    lib = _lib.load()
    nb = src.numel() * src.element_size() if nbytes is None else int(nbytes)
    ev = event.cuda_event if event is not None else None
    rc = lib.elx_copy_d2h(dst_host.data_ptr(), src.data_ptr(), nb, _stream(stream), ev)
    _lib.check(rc, "elx_copy_d2h")


def colsum(x2d: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    """K7: out[j] = sum_i x2d[i, j] (fp32 accumulation, deterministic), written
    in out's dtype — bias gradients straight into their chunk slots."""
    lib = _lib.load()
    _cuda(x2d, "x2d")
    if x2d.dim() != 2 or out.numel() != x2d.shape[1]:
        raise ValidationError("colsum needs a 2-D input and out of x2d.shape[1] elements")
    rows, cols = x2d.shape
    nws = lib.elx_colsum_workspace(rows, cols)
    # the workspace lives until the launch is enqueued, and the allocator may hand its memory out again
    # only once the launch stream has passed it (record_stream), whatever stream that is
    ws = torch.empty(nws, dtype=torch.float32, device=x2d.device) if nws > 0 else None
    st = stream if stream is not None else torch.cuda.current_stream(x2d.device)
    rc = lib.elx_colsum(out.data_ptr(), elx_dtype(out.dtype), x2d.data_ptr(), elx_dtype(x2d.dtype), rows, cols,
                        None if ws is None else ws.data_ptr(), st.cuda_stream)
    if ws is not None:
        ws.record_stream(st)
    _lib.check(rc, "elx_colsum")


def colsum_batched(xs: Sequence[torch.Tensor], outs: Sequence[torch.Tensor], stream=None) -> None:
    """K7 over up to 4 same-shape 2-D inputs in one launch: outs[i] = colsum(xs[i])."""
    lib = _lib.load()
    if not 1 <= len(xs) <= 4 or len(xs) != len(outs):
        raise ValidationError("colsum_batched takes 1..4 inputs and as many outputs")
    rows, cols = xs[0].shape
    for x, o in zip(xs, outs):
        _cuda(x, "x")
        if x.shape != (rows, cols) or x.dtype != xs[0].dtype or o.numel() != cols or o.dtype != outs[0].dtype:
            raise ValidationError("colsum_batched inputs/outputs must share shape and dtype")
    ins = _ptr_array([x.data_ptr() for x in xs])
    ots = _ptr_array([o.data_ptr() for o in outs])
    rc = lib.elx_colsum_batched(len(xs), ctypes.addressof(ots), elx_dtype(outs[0].dtype), ctypes.addressof(ins),
                                elx_dtype(xs[0].dtype), rows, cols, _stream(stream))
    _lib.check(rc, "elx_colsum_batched")


def colsum_geometry(rows: int, cols: int) -> tuple[int, int]:
    """(slices, sub-slices per slice) of K7's fixed summation order."""
    lib = _lib.load()
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.elx_colsum_geometry(int(rows), int(cols), ctypes.byref(a), ctypes.byref(b)), "elx_colsum_geometry")
    return a.value, b.value


def ln_param_grad(x2d: torch.Tensor, dy2d: torch.Tensor, mean: torch.Tensor, rstd: torch.Tensor,
                  dgamma: torch.Tensor, dbeta: torch.Tensor, stream=None) -> None:
    """K9: LayerNorm weight/bias gradients written into dgamma/dbeta (the
    chunk slots): dgamma = sum_r dy * (x - mean) * rstd, dbeta = sum_r dy
    (fp32, deterministic order)."""
    lib = _lib.load()
    for t, w in ((x2d, "x"), (dy2d, "dy"), (mean, "mean"), (rstd, "rstd")):
        _cuda(t, w)
    rows, cols = x2d.shape
    if dy2d.shape != x2d.shape or dy2d.dtype != x2d.dtype or mean.numel() != rows or rstd.numel() != rows:
        raise ValidationError("ln_param_grad: x/dy shapes or dtypes differ, or mean/rstd are not one per row")
    if mean.dtype != torch.float32 or rstd.dtype != torch.float32:
        raise ValidationError("ln_param_grad: mean/rstd must be float32")
    if dgamma.numel() != cols or dbeta.numel() != cols or dgamma.dtype != x2d.dtype or dbeta.dtype != x2d.dtype:
        raise ValidationError("ln_param_grad: dgamma/dbeta must hold `cols` elements of x's dtype")
    rc = lib.elx_ln_param_grad(dgamma.data_ptr(), dbeta.data_ptr(), x2d.data_ptr(), dy2d.data_ptr(), mean.data_ptr(),
                               rstd.data_ptr(), elx_dtype(x2d.dtype), rows, cols, _stream(stream))
    _lib.check(rc, "elx_ln_param_grad")


def layer_norm_fwd(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor, eps: float = 1e-5, stream=None):
    """K10: LayerNorm over the last dimension; returns (y, mean, rstd) with
    fp32 mean/rstd of shape x.shape[:-1] (what K9 and K11 read back)."""
    lib = _lib.load()
    for t, n in ((x, "x"), (w, "w"), (b, "b")):
        _cuda(t, n)
    H = x.shape[-1]
    if w.numel() != H or b.numel() != H or w.dtype != x.dtype or b.dtype != x.dtype:
        raise ValidationError("layer_norm_fwd: w/b must hold x.shape[-1] elements of x's dtype")
    rows = x.numel() // H
    y = torch.empty_like(x)
    mean = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    rstd = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    rc = lib.elx_layer_norm_fwd(y.data_ptr(), mean.data_ptr(), rstd.data_ptr(), x.data_ptr(), w.data_ptr(),
                                b.data_ptr(), elx_dtype(x.dtype), rows, H, float(eps), _stream(stream))
    _lib.check(rc, "elx_layer_norm_fwd")
    return y, mean, rstd


def layer_norm_bwd_dx(x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, mean: torch.Tensor, rstd: torch.Tensor,
                      dres: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """K11: the LayerNorm input gradient (the weight/bias gradients are K9's);
    with `dres` (the gradient reaching x through a residual branch) it is
    added in the same pass, bit-identical to a separate add."""
    lib = _lib.load()
    for t, n in ((x, "x"), (dy, "dy"), (w, "w"), (mean, "mean"), (rstd, "rstd")):
        _cuda(t, n)
    H = x.shape[-1]
    if dy.shape != x.shape or dy.dtype != x.dtype or mean.numel() * H != x.numel():
        raise ValidationError("layer_norm_bwd_dx: dy must match x; mean/rstd one per row")
    if dres is not None:
        _cuda(dres, "dres")
        if dres.shape != x.shape or dres.dtype != x.dtype or not dres.is_contiguous():
            raise ValidationError("layer_norm_bwd_dx: dres must be a contiguous tensor like x")
    dx = torch.empty_like(x)
    rc = lib.elx_layer_norm_bwd_dx_res(dx.data_ptr(), x.data_ptr(), dy.data_ptr(), w.data_ptr(), mean.data_ptr(),
                                       rstd.data_ptr(), None if dres is None else dres.data_ptr(),
                                       elx_dtype(x.dtype), x.numel() // H, H, _stream(stream))
    _lib.check(rc, "elx_layer_norm_bwd_dx")
    return dx


def gelu_fwd(x: torch.Tensor, stream=None) -> torch.Tensor:
    """K12: tanh-approximated GELU (the GPT-2 MLP activation)."""
    _cuda(x, "x")
    y = torch.empty_like(x)
    rc = _lib.load().elx_gelu_fwd(y.data_ptr(), x.data_ptr(), elx_dtype(x.dtype), x.numel(), _stream(stream))
    _lib.check(rc, "elx_gelu_fwd")
    return y


def gelu_bwd(x: torch.Tensor, dy: torch.Tensor, stream=None) -> torch.Tensor:
    _cuda(x, "x")
    _cuda(dy, "dy")
    if dy.shape != x.shape or dy.dtype != x.dtype:
        raise ValidationError("gelu_bwd: dy must match x")
    dx = torch.empty_like(x)
    rc = _lib.load().elx_gelu_bwd(dx.data_ptr(), x.data_ptr(), dy.data_ptr(), elx_dtype(x.dtype), x.numel(),
                                  _stream(stream))
    _lib.check(rc, "elx_gelu_bwd")
    return dx


def gelu_bwd_colsum(x2d: torch.Tensor, dy2d: torch.Tensor, dbias: torch.Tensor, stream=None) -> torch.Tensor:
    """K12 backward fused with K7: returns dx = dy * gelu'(x) and writes
    colsum(dx) into `dbias` (bit-identical to gelu_bwd + colsum)."""
    _cuda(x2d, "x")
    _cuda(dy2d, "dy")
    if x2d.dim() != 2 or dy2d.shape != x2d.shape or dy2d.dtype != x2d.dtype or dbias.numel() != x2d.shape[1]:
        raise ValidationError("gelu_bwd_colsum: x, dy [rows, cols] of one dtype; dbias of cols elements")
    dx = torch.empty_like(x2d)
    rows, cols = x2d.shape
    rc = _lib.load().elx_gelu_bwd_colsum(dx.data_ptr(), dbias.data_ptr(), elx_dtype(dbias.dtype), x2d.data_ptr(),
                                         dy2d.data_ptr(), elx_dtype(x2d.dtype), rows, cols, _stream(stream))
    _lib.check(rc, "elx_gelu_bwd_colsum")
    return dx


def embedding_bwd(grad_w: torch.Tensor, tokens: torch.Tensor, dy2d: torch.Tensor, stream=None) -> None:
    """K13: grad_w[t] += sum of dy rows at the positions of token t (fp32 sum
    in position order, rounded once, then added) — deterministic, in place.
    grad_w [rows, H] (row stride may exceed H), tokens int64 [n], dy2d [n, H]."""
    if not grad_w.is_cuda:
        raise ValidationError("grad_w must be a CUDA tensor")
    _cuda(dy2d, "dy")
    n, H = dy2d.shape
    if grad_w.dim() != 2 or grad_w.shape[1] != H or grad_w.stride(1) != 1 or grad_w.dtype != dy2d.dtype \
            or not dy2d.is_contiguous() or tokens.numel() != n:
        raise ValidationError("embedding_bwd: grad_w [rows, H] (unit column stride), dy [n, H] contiguous, n tokens")
    sorted_tok, perm = torch.sort(tokens.reshape(-1), stable=True)
    rc = _lib.load().elx_embedding_bwd(grad_w.data_ptr(), grad_w.stride(0), dy2d.data_ptr(), sorted_tok.data_ptr(),
                                       perm.data_ptr(), n, H, elx_dtype(dy2d.dtype), _stream(stream))
    _lib.check(rc, "elx_embedding_bwd")


class LMHeadCrossEntropy(torch.autograd.Function):
    """K8: mean softmax cross-entropy over the padded bf16/f16 lm_head logits
    [rows, ld] (columns >= vocab excluded), with no fp32 copy of the logits.
    Forward: per-row log-sum-exp and loss (elx_xent_fwd), mean over counted
    rows. Backward: the logits buffer is overwritten in place by its gradient
    (elx_xent_bwd) — the GEMM that produced it does not need it back — scaled
    on the device by upstream / count. Matches F.cross_entropy(logits[:, :vocab]
    .float(), targets) within float32 tolerance (tests/test_kernels_gpu.py)."""

    @staticmethod
    def forward(ctx, logits: torch.Tensor, targets: torch.Tensor, vocab: int, ignore_index: int = -100):
        lib = _lib.load()
        _cuda(logits, "logits")
        if logits.dim() != 2 or logits.dtype not in (torch.bfloat16, torch.float16):
            raise ValidationError("logits must be a contiguous 2-D bf16/f16 tensor")
        rows, ld = logits.shape
        tg = targets.reshape(-1)
        if tg.numel() != rows or tg.dtype != torch.int64 or not tg.is_cuda:
            raise ValidationError("targets must be int64 CUDA with one entry per logits row")
        tg = tg.contiguous()
        lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
        loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
        rc = lib.elx_xent_fwd(logits.data_ptr(), elx_dtype(logits.dtype), rows, ld, int(vocab), tg.data_ptr(), int(ignore_index),
                              lse.data_ptr(), loss.data_ptr(), _stream(None))
        _lib.check(rc, "elx_xent_fwd")
        count = (tg != ignore_index).sum().to(torch.float32)
        ctx.save_for_backward(logits, tg, lse, count)
        ctx.vocab, ctx.ignore = int(vocab), int(ignore_index)
        return loss.sum() / count

    @staticmethod
    def backward(ctx, g):
        logits, tg, lse, count = ctx.saved_tensors
        rows, ld = logits.shape
        scale = (g.to(torch.float32) / count).reshape(1).contiguous()
        rc = _lib.load().elx_xent_bwd(logits.data_ptr(), elx_dtype(logits.dtype), rows, ld, ctx.vocab, tg.data_ptr(), ctx.ignore,
                                      lse.data_ptr(), scale.data_ptr(), _stream(None))
        _lib.check(rc, "elx_xent_bwd")
        return logits, None, None, None


def lm_head_cross_entropy(logits: torch.Tensor, targets: torch.Tensor, vocab: int, ignore_index: int = -100):
    return LMHeadCrossEntropy.apply(logits, targets, vocab, ignore_index)


# ------------------------------------------------------------------ cuBLASLt GEMMs with fused epilogues
EPI_NONE, EPI_BIAS, EPI_GELU_BIAS, EPI_GELU_AUX_BIAS, EPI_DGELU_BGRAD, EPI_BGRADB = range(6)
_LT_WS: dict = {}
_LT_WS_BYTES = 32 * 2 ** 20


def _lt_workspace(device: torch.device) -> int:
    """One cuBLASLt workspace per (device, host thread). A thread issues its
    GEMMs on one stream at a time (eager steps and graph replays are ordered
    on the current stream), so its calls never overlap; ranks run as threads
    on one GPU (tests/_refstep.py, scripts/emulate_ranks.py) get their own,
    since split-K scratch shared between concurrent streams would race.
    Allocated on first use, which capture() guarantees happens before a graph
    capture (its warm-up steps run eagerly on the same thread), so the
    captured pointer is ordinary device memory, not the graph's pool."""
    key = (device.index, threading.get_ident())
    ws = _LT_WS.get(key)
    if ws is None:
        ws = torch.empty(_LT_WS_BYTES, dtype=torch.uint8, device=device)
        _LT_WS[key] = ws
    return ws.data_ptr()


# Per-shape cuBLASLt algorithm choice: index into the heuristic's candidate
# list, tuned once on the B200 by scripts/tune_lt.py (fastest with L2 flushed,
# median of repeats) and committed, so every process picks the same algorithm.
# Shapes not in the table take the heuristic's first candidate.
_LT_TABLE_PATH = Path(__file__).resolve().parents[1] / "plans" / "lt_algos_b200.json"
_LT_TABLE: dict | None = None
LT_RECORD: set | None = None  # scripts/tune_lt.py collects the step's GEMM keys here


def lt_key(epi, dt, ta, tb, m, n, k, lda, ldb, ldd, ldaux, has_c) -> tuple:
    return (int(epi), int(dt), int(ta), int(tb), int(m), int(n), int(k), int(lda), int(ldb), int(ldd), int(ldaux),
            int(bool(has_c)))


def _lt_table() -> dict:
    """The tuned table, used only on the GPU model it was tuned on (on other
    hardware every shape takes the heuristic's first candidate)."""
    global _LT_TABLE
    if _LT_TABLE is None:
        table = {}
        if os.environ.get("ELX_LT_TABLE", "1") != "0" and _LT_TABLE_PATH.exists():
            doc = json.loads(_LT_TABLE_PATH.read_text())
            gpu = torch.cuda.get_device_name() if torch.cuda.is_available() else doc.get("gpu")
            if doc.get("gpu") == gpu:
                for rec in doc["choices"]:
                    table[tuple(rec["key"])] = int(rec["index"])
        _LT_TABLE = table
    return _LT_TABLE


def _lt(epi, ta, tb, m, n, k, a, lda, b, ldb, d, ldd, bias=None, aux=None, ldaux=0, stream=None, c=None,
        algo=None):
    lib = _lib.load()
    dt = elx_dtype(d.dtype)
    key = lt_key(epi, dt, ta, tb, m, n, k, lda, ldb, ldd, ldaux, c is not None)
    if LT_RECORD is not None:
        LT_RECORD.add(key)
    idx = _lt_table().get(key, -1) if algo is None else algo
    args = (epi, dt, ta, tb, m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, None if c is None else c.data_ptr(),
            d.data_ptr(), ldd, None if bias is None else bias.data_ptr(), None if aux is None else aux.data_ptr(),
            ldaux, _lt_workspace(d.device), _LT_WS_BYTES)
    rc = lib.elx_lt_matmul_ex(*args, idx, _stream(stream))
    if rc == _lib.ERR_VALIDATION and algo is None and idx > 0:
        # the table's index is past this library's candidate list (another cuBLASLt): drop the entry
        _lt_table().pop(key, None)
        rc = lib.elx_lt_matmul_ex(*args, -1, _stream(stream))
    _lib.check(rc, "elx_lt_matmul")


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, *, ta: bool = False, tb: bool = False,
         bias: torch.Tensor | None = None, c: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Row-major out[M, N] = op(a) @ op(b) (+ c) (+ bias[N]) through
    elx_lt_matmul (op = transpose when ta / tb); 2-D contiguous operands."""
    for t, n in ((a, "a"), (b, "b")):
        _cuda(t, n)
        if t.dim() != 2 or not t.is_contiguous():
            raise ValidationError(f"gemm: {n} must be a contiguous 2-D tensor")
    M, K = (a.shape[1], a.shape[0]) if ta else a.shape
    K2, N = (b.shape[1], b.shape[0]) if tb else b.shape
    if K != K2:
        raise ValidationError(f"gemm: inner dimensions {K} and {K2} differ")
    if out is None:
        out = torch.empty(M, N, dtype=a.dtype, device=a.device)
    if out.shape != (M, N) or not out.is_contiguous():
        raise ValidationError("gemm: out must be a contiguous [M, N] tensor")
    # column-major: out^T [N, M] = op(b)^T [N, K] . op(a)^T [K, M]
    _lt(EPI_BIAS if bias is not None else EPI_NONE, 1 if tb else 0, 1 if ta else 0, N, M, K, b, b.shape[1], a,
        a.shape[1], out, N, bias=bias, c=c, stream=stream)
    return out


def linear_gelu(x2d: torch.Tensor, w: torch.Tensor, b: torch.Tensor, keep_aux: bool, stream=None):
    """gelu(x W^T + b) in one GEMM (tanh-GELU epilogue); with keep_aux also the
    pre-activation x W^T + b the backward needs. x2d [T, I], w [O, I], b [O]."""
    T, I = x2d.shape
    O = w.shape[0]
    for t, n in ((x2d, "x"), (w, "w"), (b, "b")):
        _cuda(t, n)
    y = torch.empty(T, O, dtype=x2d.dtype, device=x2d.device)
    aux = torch.empty(T, O, dtype=x2d.dtype, device=x2d.device) if keep_aux else None
    # column-major: y^T [O, T] = W [O, I] . x^T [I, T]
    _lt(EPI_GELU_AUX_BIAS if keep_aux else EPI_GELU_BIAS, 1, 0, O, T, I, w, I, x2d, I, y, O, bias=b, aux=aux,
        ldaux=O if keep_aux else 0, stream=stream)
    return y, aux


def linear_dgelu_bgrad(dy2d: torch.Tensor, w: torch.Tensor, pre: torch.Tensor, dbias: torch.Tensor, stream=None):
    """For y = gelu(pre) W^T + c: d_pre = (dy W) * gelu'(pre) in one GEMM, and
    the bias gradient of `pre` (= colsum of d_pre) written into `dbias`.
    dy2d [T, O], w [O, I], pre [T, I], dbias [I]."""
    T, O = dy2d.shape
    I = w.shape[1]
    for t, n in ((dy2d, "dy"), (w, "w"), (pre, "pre"), (dbias, "dbias")):
        _cuda(t, n)
    d = torch.empty(T, I, dtype=dy2d.dtype, device=dy2d.device)
    # column-major: d^T [I, T] = W^T [I, O] . dy^T [O, T]
    _lt(EPI_DGELU_BGRAD, 0, 0, I, T, O, w, I, dy2d, O, d, I, bias=dbias, aux=pre, ldaux=I, stream=stream)
    return d


def wgrad_bgrad(x2d: torch.Tensor, dy2d: torch.Tensor, dw: torch.Tensor, db: torch.Tensor | None, stream=None):
    """dW = dy^T x written into `dw` [O, I] and (db given) db = colsum(dy) from
    the same GEMM's epilogue. x2d [T, I], dy2d [T, O]."""
    T, I = x2d.shape
    O = dy2d.shape[1]
    for t, n in ((x2d, "x"), (dy2d, "dy"), (dw, "dw")):
        _cuda(t, n)
    # column-major: dW^T [I, O] = x^T [I, T] . dy [T, O]
    _lt(EPI_BGRADB if db is not None else EPI_NONE, 0, 1, I, O, T, x2d, I, dy2d, O, dw, I, bias=db, stream=stream)


def linear_residual(x2d: torch.Tensor, w: torch.Tensor, b: torch.Tensor, res2d: torch.Tensor, stream=None):
    """res + x W^T + b in one GEMM (C operand + bias epilogue): the residual add
    of an output projection without a separate elementwise pass.
    x2d [T, I], w [O, I], b [O], res2d [T, O]."""
    T, I = x2d.shape
    O = w.shape[0]
    for t, n in ((x2d, "x"), (w, "w"), (b, "b"), (res2d, "res")):
        _cuda(t, n)
    if res2d.shape != (T, O) or res2d.dtype != x2d.dtype:
        raise ValidationError("linear_residual: res must be [T, O] of x's dtype")
    y = torch.empty(T, O, dtype=x2d.dtype, device=x2d.device)
    # column-major: y^T [O, T] = W [O, I] . x^T [I, T] + res^T
    _lt(EPI_BIAS, 1, 0, O, T, I, w, I, x2d, I, y, O, bias=b, c=res2d, stream=stream)
    return y
