"""GPT-2 training step driven through the chunk runtime (the path's caller).

Every coarse node of the access trace (profiles.py:490-521: wpe embed, one
node per AC-grouped layer, ln_f, the tied lm_head) is a "wrapped operator"
(PAPER.md:203-206): before it runs, the ChunkFetcher makes its chunks
resident. With activation checkpointing (recompute=True)
the forward saves only each node's input and the backward recomputes each
node with autograd; when no chunk can leave its block between a node's
forward and backward, recompute="auto"/False keeps the forward's autograd
graph instead (same results). The backward walks the nodes in reverse
(chunking.py:165), writes the parameter gradients over the parameter data in
the chunk and releases chunks at their reduce positions
(rcache_sim.py:160-167, K3). After the walk HybridAdam updates the shards.

GEMMs are cuBLASLt through elx_lt_matmul_ex (fused epilogues: the MLP's bias
+ GELU, the output projections' residual add; a per-shape algorithm table
tuned on the B200), attention is torch SDPA (cuDNN); LayerNorm, GELU, the
lm_head cross-entropy, the embedding gradient and every gradient reduction
written into the chunk are our kernels (csrc/elx_model_kernels.cu), and the
chunk path itself is ours (csrc/elx_kernels.cu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import kernels
from .errors import ValidationError
from .layout import build_chunk_trace, pack_chunks
from .profiles import coarsen_graph, partition_multiuse, synthesize_transformer_profile
from .runtime import ChunkFetcher, ChunkManager, HybridAdam, LossScaler
from .schedule import as_plan
from .transport import make_transport


@dataclass(frozen=True)
class GPT2Config:
    hidden: int
    layers: int
    heads: int
    vocab: int = 50257
    seq_len: int = 1024
    batch: int = 8

    @property
    def name(self) -> str:
        return f"gpt2-h{self.hidden}-l{self.layers}"

    @property
    def vocab_padded(self) -> int:
        """Vocab rounded up to 64 rows for the lm_head GEMMs only: an odd
        leading dimension (50257) forces cuBLAS onto align-1 kernels (3x
        slower on the lm_head). The parameter keeps vocab*hidden elements;
        the pad rows are zero and receive no update."""
        return -(-self.vocab // 64) * 64


PRESETS = {  # BASELINE.json configs; Table 7 shapes
    "gpt2-small": GPT2Config(768, 12, 12),
    "gpt2-1.3b": GPT2Config(2048, 24, 16),
    "gpt2-4b": GPT2Config(3072, 32, 24),
    "gpt2-10b": GPT2Config(4096, 48, 32),
}


def param_shapes(cfg: GPT2Config) -> dict[str, tuple[int, ...]]:
    h = cfg.hidden
    shapes = {"wte": (cfg.vocab, h), "wpe": (cfg.seq_len, h), "ln_f.w": (h,), "ln_f.b": (h,)}
    for i in range(cfg.layers):
        p = f"h{i}."
        shapes.update({
            p + "ln_1.w": (h,), p + "ln_1.b": (h,),
            p + "attn.qkv.w": (3 * h, h), p + "attn.qkv.b": (3 * h,),
            p + "attn.proj.w": (h, h), p + "attn.proj.b": (h,),
            p + "ln_2.w": (h,), p + "ln_2.b": (h,),
            p + "mlp.fc.w": (4 * h, h), p + "mlp.fc.b": (4 * h,),
            p + "mlp.proj.w": (h, 4 * h), p + "mlp.proj.b": (h,),
        })
    return shapes


def init_params(cfg: GPT2Config, device, seed: int = 1234, dtype=torch.bfloat16) -> dict[str, torch.Tensor]:
    """N(0, 0.02) weights, LN weight 1, biases 0."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = {}
    for pid, shp in param_shapes(cfg).items():
        if pid.endswith(".b"):
            out[pid] = torch.zeros(shp, dtype=dtype, device=device)
        elif "ln_" in pid:
            out[pid] = torch.ones(shp, dtype=dtype, device=device)
        else:
            out[pid] = (torch.randn(shp, generator=g, device=device, dtype=torch.float32) * 0.02).to(dtype)
    return out


def layer_pieces(i: int, h: int) -> list[tuple[str, int, tuple[int, ...]]]:
    """The tensors one layer computes with, as (param id, element offset in
    the parameter, shape). attn.qkv.w/.b are used as three row blocks (q, k,
    v): each projection's output is then contiguous [B, T, H], its
    [B, heads, T, hd] view is dense, SDPA's backward returns dq/dk/dv in that
    same dense layout, and no stack/permute copy is needed in the backward
    (6.0 + 3.4 ms of a 104 ms step before, profiles/r01b_launches.md)."""
    p = f"h{i}."
    out = [(p + "ln_1.w", 0, (h,)), (p + "ln_1.b", 0, (h,))]
    out += [(p + "attn.qkv.w", j * h * h, (h, h)) for j in range(3)]
    out += [(p + "attn.qkv.b", j * h, (h,)) for j in range(3)]
    out += [(p + "attn.proj.w", 0, (h, h)), (p + "attn.proj.b", 0, (h,)),
            (p + "ln_2.w", 0, (h,)), (p + "ln_2.b", 0, (h,)),
            (p + "mlp.fc.w", 0, (4 * h, h)), (p + "mlp.fc.b", 0, (4 * h,)),
            (p + "mlp.proj.w", 0, (h, 4 * h)), (p + "mlp.proj.b", 0, (h,))]
    return out


class _Embedding(torch.autograd.Function):
    """The token embedding lookup wte[tokens]. Backward: K13 accumulates the
    gradient into `w_target` (the shared wte gradient buffer, [vocab, H],
    already holding the tied head's part) in place; without a target it
    returns a dense gradient made by the same kernel over zeros — so both
    paths give the same bits."""

    @staticmethod
    def forward(ctx, tokens, wte, w_target):
        ctx.save_for_backward(tokens)
        ctx.wshape, ctx.target = wte.shape, w_target
        return F.embedding(tokens, wte)

    @staticmethod
    def backward(ctx, gy):
        (tokens,) = ctx.saved_tensors
        gy2 = gy.reshape(-1, gy.shape[-1]).contiguous()
        if ctx.target is None:
            dw = torch.zeros(ctx.wshape, dtype=gy.dtype, device=gy.device)
            kernels.embedding_bwd(dw, tokens, gy2)
            return None, dw, None
        kernels.embedding_bwd(ctx.target, tokens, gy2)
        return None, None, None


class _TiedHead(torch.autograd.Function):
    """logits = x wte^T over the padded vocab rows (the tied lm_head), GEMMs
    through elx_lt_matmul_ex. Backward: dX = dlogits wte; dW = dlogits^T x
    over the `vocab` real rows only — written straight into `w_target` (the
    shared wte gradient buffer, [vocab, H]) when given, so no padded gradient
    tensor and no K1 copy exist; without a target it is returned (padded)."""

    @staticmethod
    def forward(ctx, x2, wte, vocab, w_target):
        ctx.save_for_backward(x2, wte)
        ctx.vocab, ctx.target = int(vocab), w_target
        return kernels.gemm(x2.contiguous(), wte, tb=True)

    @staticmethod
    def backward(ctx, gl):
        x2, wte = ctx.saved_tensors
        gl = gl.contiguous()
        T, Vp = gl.shape
        H = x2.shape[1]
        gx = kernels.gemm(gl, wte) if ctx.needs_input_grad[0] else None
        dw = torch.zeros_like(wte) if ctx.target is None else None
        tgt = ctx.target if dw is None else dw[:ctx.vocab]
        # column-major: dW^T [H, vocab] = x^T [H, T] . dlogits[:, :vocab] [T, vocab] (ld = Vp); the same
        # call (same algorithm) with or without a target, so both give the same bits
        kernels._lt(kernels.EPI_NONE, 0, 1, H, ctx.vocab, T, x2, H, gl, Vp, tgt, H)
        return gx, dw, None, None


def _qkv_proj(h, wq, wk, wv, bq, bk, bv):
    """q, k, v = h W^T + b for the three row blocks of attn.qkv as ONE GEMM
    with N = 3H (the blocks are consecutive in the chunk, so W and b are one
    strided view each). The outputs are [B, T, H] column blocks of one
    [B, T, 3H] result; SDPA takes them strided at the same speed (0.136 vs
    0.146 ms for three N = H GEMMs at the 1.3B shape, scripts/qkv_probe.py)."""
    H = wq.shape[1]
    es = wq.element_size()
    same = (wq.untyped_storage().data_ptr() == wk.untyped_storage().data_ptr() == wv.untyped_storage().data_ptr()
            and bq.untyped_storage().data_ptr() == bk.untyped_storage().data_ptr() == bv.untyped_storage().data_ptr())
    packed = same and (wk.data_ptr() == wq.data_ptr() + wq.numel() * es and wv.data_ptr() == wk.data_ptr() + wk.numel() * es
              and bk.data_ptr() == bq.data_ptr() + bq.numel() * es and bv.data_ptr() == bk.data_ptr() + bk.numel() * es
              and wq.is_contiguous() and wk.is_contiguous() and wv.is_contiguous())
    if not packed:
        return F.linear(h, wq, bq), F.linear(h, wk, bk), F.linear(h, wv, bv)
    n = wq.shape[0] + wk.shape[0] + wv.shape[0]
    y = kernels.gemm(h.reshape(-1, H).contiguous(), wq.as_strided((n, H), (H, 1)), tb=True,
                     bias=bq.as_strided((n,), (1,))).view(*h.shape[:-1], n)
    a, b = wq.shape[0], wq.shape[0] + wk.shape[0]
    return y[..., :a], y[..., a:b], y[..., b:]


class _OverwriteQKV(torch.autograd.Function):
    """The three attention input projections q/k/v = h W^T + b as ONE wrapped
    operator (three row blocks of attn.qkv, each output dense for SDPA). Its
    backward accumulates dH = dq Wq + dk Wk + dv Wv in the GEMMs (beta = 1, no
    separate add kernels), writes the three weight gradients into their row
    blocks of the chunk slot, and the three bias gradients with ONE batched K7
    launch."""

    @staticmethod
    def forward(ctx, h, wq, wk, wv, bq, bk, bv, tq, tk, tv, sq, sk, sv):
        ctx.save_for_backward(h, wq, wk, wv)
        ctx.targets = (tq, tk, tv, sq, sk, sv)
        return _qkv_proj(h, wq, wk, wv, bq, bk, bv)

    @staticmethod
    def backward(ctx, gq, gk, gv):
        h, wq, wk, wv = ctx.saved_tensors
        tq, tk, tv, sq, sk, sv = ctx.targets
        H = h.shape[-1]
        gs = [g.reshape(-1, g.shape[-1]).contiguous() for g in (gq, gk, gv)]
        h2 = h.reshape(-1, H).contiguous()
        gh = None
        if ctx.needs_input_grad[0]:
            gh = kernels.gemm(gs[0], wq)
            kernels.gemm(gs[1], wk, out=gh, c=gh)  # accumulated in the GEMM (beta = 1)
            kernels.gemm(gs[2], wv, out=gh, c=gh)
            gh = gh.view(h.shape)
        for g, t in zip(gs, (tq, tk, tv)):
            kernels.gemm(g, h2, ta=True, out=t)
        kernels.colsum_batched(gs, (sq, sk, sv))
        return (gh,) + (None,) * 12


class _OverwriteLinearResidual(torch.autograd.Function):
    """y = res + x W^T + b as ONE cuBLASLt GEMM (C operand + bias epilogue):
    an output projection (attn.proj, mlp.proj) with the residual add folded in.
    Backward: dX first (W intact), then dW by a GEMM straight into the
    weight's chunk slot and db by K7 into the bias slot — the gradient
    overwrites the parameter data (Fig. 3) with no gradient
    tensor and no K1 copy; the residual's gradient is dy itself."""

    @staticmethod
    def forward(ctx, x, w, b, res, w_target, b_target):
        x2 = x.reshape(-1, x.shape[-1])
        y = kernels.linear_residual(x2, w, b, res.reshape(-1, w.shape[0]))
        ctx.save_for_backward(x2, w)
        ctx.targets = (w_target, b_target)
        ctx.xshape = x.shape
        return y.view(res.shape)

    @staticmethod
    def backward(ctx, gy):
        x2, w = ctx.saved_tensors
        w_t, b_t = ctx.targets
        gy2 = gy.reshape(-1, gy.shape[-1])
        gy2 = gy2.contiguous()
        gx = kernels.gemm(gy2, w).view(ctx.xshape) if ctx.needs_input_grad[0] else None
        kernels.gemm(gy2, x2, ta=True, out=w_t)
        kernels.colsum(gy2, b_t)
        return gx, None, None, gy, None, None


class _LayerNorm(torch.autograd.Function):
    """LayerNorm over the last dimension (eps 1e-5) on our kernels: forward
    K10 (y plus the fp32 mean/rstd), backward K11 for dX and K9 for dW/db.
    With `targets` (chunk slots) the weight/bias gradients are written
    straight over the parameter data and no gradient
    tensor is returned for them: no GammaBeta kernel, no K1 write-back."""

    @staticmethod
    def forward(ctx, x, w, b, w_target, b_target):
        x = x.contiguous()
        y, mean, rstd = kernels.layer_norm_fwd(x, w, b)
        ctx.save_for_backward(x, w, mean, rstd)
        ctx.targets = (w_target, b_target)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, w, mean, rstd = ctx.saved_tensors
        H = x.shape[-1]
        gy = gy.contiguous()
        gx = kernels.layer_norm_bwd_dx(x, gy, w, mean, rstd)
        w_t, b_t = ctx.targets
        own = w_t is None
        if own:
            w_t, b_t = torch.empty_like(w), torch.empty_like(w)
        kernels.ln_param_grad(x.reshape(-1, H), gy.reshape(-1, H), mean.reshape(-1), rstd.reshape(-1), w_t, b_t)
        return gx, (w_t if own else None), (b_t if own else None), None, None


class _LayerNormResidual(torch.autograd.Function):
    """_LayerNorm for an x that also feeds a residual branch: returns (y, x')
    with x' an alias of x for the residual. The two gradients reaching x (the
    LayerNorm's and the residual's) are summed inside K11's store instead of
    by autograd's separate add kernel over [T, H] (bit-identical)."""

    @staticmethod
    def forward(ctx, x, w, b, w_target, b_target):
        x = x.contiguous()
        y, mean, rstd = kernels.layer_norm_fwd(x, w, b)
        ctx.save_for_backward(x, w, mean, rstd)
        ctx.targets = (w_target, b_target)
        return y, x.view_as(x)

    @staticmethod
    def backward(ctx, gy, gres):
        x, w, mean, rstd = ctx.saved_tensors
        H = x.shape[-1]
        gy = gy.contiguous()
        gx = kernels.layer_norm_bwd_dx(x, gy, w, mean, rstd, dres=None if gres is None else gres.contiguous())
        w_t, b_t = ctx.targets
        own = w_t is None
        if own:
            w_t, b_t = torch.empty_like(w), torch.empty_like(w)
        kernels.ln_param_grad(x.reshape(-1, H), gy.reshape(-1, H), mean.reshape(-1), rstd.reshape(-1), w_t, b_t)
        return gx, (w_t if own else None), (b_t if own else None), None, None


def layer_norm_residual(x, w, b, w_target=None, b_target=None):
    """(layer_norm(x), x) where the returned x feeds a residual branch; under
    autograd the two gradients of x are joined inside K11."""
    if torch.is_grad_enabled() and (x.requires_grad or w.requires_grad or b.requires_grad):
        return _LayerNormResidual.apply(x, w, b, w_target, b_target)
    return kernels.layer_norm_fwd(x.contiguous(), w, b)[0], x


def layer_norm(x, w, b, w_target=None, b_target=None):
    """GPT-2 LayerNorm on K10/K11/K9 (autograd only when a gradient is needed)."""
    if torch.is_grad_enabled() and (x.requires_grad or w.requires_grad or b.requires_grad):
        return _LayerNorm.apply(x, w, b, w_target, b_target)
    return kernels.layer_norm_fwd(x.contiguous(), w, b)[0]


class _OverwriteFcGelu(torch.autograd.Function):
    """a = gelu(x W^T + b), the MLP's first wrapped operator, as ONE cuBLASLt
    GEMM with the bias + tanh-GELU epilogue (keeping the pre-activation for the
    backward): the separate GELU pass over the [T, 4H] activation disappears.
    Backward: K12's GELU derivative fused with K7's column sum (db straight
    into the bias slot) in one pass, dW by cuBLAS into the
    weight slot, dX by cuBLAS. (cuBLASLt's fused
    DGELU_BGRAD and BGRADB epilogues measured slower on B200 than this
    sequence: 0.62 vs 0.26 ms and 62 vs 60 us, profiles/r01o_model_kernels.jsonl.)"""

    @staticmethod
    def forward(ctx, x, w, b, w_target, b_target):
        x2 = x.reshape(-1, x.shape[-1])
        y, pre = kernels.linear_gelu(x2, w, b, keep_aux=True)
        ctx.save_for_backward(x2, w, pre)
        ctx.targets = (w_target, b_target)
        ctx.xshape = x.shape
        return y.view(*x.shape[:-1], w.shape[0])

    @staticmethod
    def backward(ctx, gy):
        x2, w, pre = ctx.saved_tensors
        w_t, b_t = ctx.targets
        d = kernels.gelu_bwd_colsum(pre, gy.reshape(-1, gy.shape[-1]).contiguous(), b_t)  # db in the same pass
        gx = kernels.gemm(d, w).view(ctx.xshape) if ctx.needs_input_grad[0] else None
        kernels.gemm(d, x2, ta=True, out=w_t)
        return gx, None, None, None, None


def fc_gelu(x, w, b, w_target=None, b_target=None):
    """gelu(x W^T + b) as one GEMM with a fused epilogue (K12 derivative in the backward)."""
    if w_target is not None:
        return _OverwriteFcGelu.apply(x, w, b, w_target, b_target)
    y, _ = kernels.linear_gelu(x.reshape(-1, x.shape[-1]), w, b, keep_aux=False)
    return y.view(*x.shape[:-1], w.shape[0])


def _alias(t: torch.Tensor) -> torch.Tensor:
    """Same storage, own version counter. Gradient targets are aliases of the
    chunk slots: every parameter of a chunk is a view of ONE storage, so an
    `out=` write through a plain view would bump the version counter shared by
    all of them and trip autograd's saved-tensor check for the (disjoint,
    still intact) parameters other operators saved."""
    a = torch.empty(0, dtype=t.dtype, device=t.device)
    return a.set_(t.untyped_storage(), t.storage_offset(), t.size(), t.stride())


# (weight, bias) positions of the six linear operators in a layer's pieces
_LINEARS = ((2, 5), (3, 6), (4, 7), (8, 9), (12, 13), (14, 15))


def _block(x, p, heads, targets=None):
    """One GPT-2 layer on its 16 compute pieces (layer_pieces order). With
    `targets` (per-piece gradient destinations) the linear operators write
    their parameter gradients there during backward."""
    B, T, H = x.shape
    hd = H // heads

    def ln(inp, wi, bi):  # (LayerNorm(inp), inp for the residual branch)
        if targets is None:
            return layer_norm_residual(inp, p[wi], p[bi])
        return layer_norm_residual(inp, p[wi], p[bi], targets[wi], targets[bi])

    def lin_res(inp, res, wi, bi):  # res + inp W^T + b, the residual add folded into the GEMM
        if targets is None:
            return kernels.linear_residual(inp.reshape(-1, inp.shape[-1]), p[wi], p[bi],
                                           res.reshape(-1, res.shape[-1])).view(res.shape)
        return _OverwriteLinearResidual.apply(inp, p[wi], p[bi], res, targets[wi], targets[bi])

    # pieces: 0/1 ln_1, 2-4 q/k/v weight blocks, 5-7 their biases, 8/9 attn.proj, 10/11 ln_2,
    # 12/13 mlp.fc, 14/15 mlp.proj (layer_pieces order)
    h, x = ln(x, 0, 1)
    if targets is None:
        qkv = _qkv_proj(h, p[2], p[3], p[4], p[5], p[6], p[7])
    else:
        qkv = _OverwriteQKV.apply(h, p[2], p[3], p[4], p[5], p[6], p[7],
                                  targets[2], targets[3], targets[4], targets[5], targets[6], targets[7])
    q, k, v = (t.view(B, T, heads, hd).transpose(1, 2) for t in qkv)
    a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    x = lin_res(a.transpose(1, 2).reshape(B, T, H), x, *_LINEARS[3])
    h, x = ln(x, 10, 11)
    fi, bi = _LINEARS[4]
    a = fc_gelu(h, p[fi], p[bi]) if targets is None else fc_gelu(h, p[fi], p[bi], targets[fi], targets[bi])
    return lin_res(a, x, *_LINEARS[5])


class ElixirGPT2:
    """Public entry point: a chunked GPT-2 trainer on one rank.

    ``plan`` is the reference planner's Plan (object or JSON text) for this
    model at this world size; ``transport`` defaults to torch.distributed
    when it is initialised with more than one rank.
    """

    def __init__(self, cfg: GPT2Config, plan, *, device=None, dtype=torch.bfloat16, seed: int = 1234,
                 lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.01,
                 max_norm: float | None = 1.0, loss_scale: float | None = None, transport=None,
                 prefetch: bool = True, cpu_threads: int | None = None, init: dict | None = None,
                 overlap_update: bool = False, cpu_update: str = "split", recompute=True):
        import torch.distributed as dist

        self.cfg = cfg
        self.device = torch.device(device if device is not None else "cuda")
        if transport is None:
            world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
            transport = make_transport(world)
        self.transport = transport
        self.profile = synthesize_transformer_profile(cfg.hidden, cfg.layers, cfg.heads, cfg.vocab,
                                                      cfg.seq_len, cfg.batch, name=cfg.name)
        self.access = coarsen_graph(self.profile)
        _, seq = partition_multiuse(self.profile)
        plan = as_plan(plan)
        self.layout = pack_chunks(seq, plan.chunk_length)
        self.trace = build_chunk_trace(self.access, self.layout)
        self.shapes = param_shapes(cfg)
        self.manager = ChunkManager(self.profile, self.layout, plan, shapes=self.shapes, transport=transport,
                                    device=self.device, dtype=dtype,
                                    shared_padded={"wte": (cfg.vocab_padded, cfg.hidden)})
        self.manager.load_params(init if init is not None else init_params(cfg, self.device, seed, dtype))
        if loss_scale is None:
            self.scaler = LossScaler(1.0, dynamic=False) if dtype == torch.bfloat16 else LossScaler(65536.0)
        else:
            self.scaler = LossScaler(loss_scale, dynamic=False)
        self.fetcher = ChunkFetcher(self.manager, self.trace, prefetch=prefetch,
                                    inv_scale=1.0 / self.scaler.scale)
        self.optimizer = HybridAdam(self.manager, lr=lr, betas=betas, eps=eps, weight_decay=weight_decay,
                                    max_norm=max_norm, cpu_threads=cpu_threads, overlap=overlap_update,
                                    cpu_update=cpu_update)
        self.optimizer.attach_fetcher(self.fetcher)
        # coarse node -> its chunk parameters, in declaration order
        order = {p.id: i for i, p in enumerate(self.profile.parameters)}
        self.node_params = [sorted(node, key=order.__getitem__) for node in self.access.coarse_ops]
        self.K = len(self.node_params)
        # compute tensors per node: (param id, element offset, shape)
        self.node_pieces = []
        for i, pids in enumerate(self.node_params):
            if 0 < i < self.K - 2:
                self.node_pieces.append(layer_pieces(i - 1, cfg.hidden))
            else:
                self.node_pieces.append([(pid, 0, self.shapes[pid]) for pid in pids])
        self.wte = self.manager.shared["wte"]
        self.last_loss = None
        self.keep_graph = self._resolve_recompute(recompute)

    def _resolve_recompute(self, recompute) -> bool:
        """Whether the forward keeps each node's autograd graph (no recompute
        in the backward) instead of activation checkpointing (PAPER.md:145-150,
        the reference's design and the default). Keeping it is valid only when
        no chunk can leave its block between a node's forward and backward —
        every rCache block stays put (n_block >= n_chunks: the schedule never
        evicts; at world 1 with every chunk GPU-home the chunks are used in
        place) — because the saved tensors are views of the chunk storage;
        "auto" also requires the activations (~17 B*T*H elements per layer)
        to fit in half the HBM left after the chunk store."""
        if recompute is True:
            return False
        m = self.manager
        resident = (m.world == 1 and not m.cpu_ids) or m.plan.n_block >= m.n_chunks  # world 1 GPU-home: in place
        if recompute is False:
            if not resident:
                raise ValidationError("recompute=False needs every chunk resident (n_block >= n_chunks)")
            return True
        if recompute != "auto":
            raise ValidationError("recompute must be True, False or 'auto'")
        cfg = self.cfg
        act = cfg.layers * 17 * cfg.batch * cfg.seq_len * cfg.hidden * self.manager.p16.element_size()
        free, _ = torch.cuda.mem_get_info(self.device)
        return resident and act < 0.5 * free

    # -------------------------------------------------------------- nodes
    def _run_node(self, i: int, x, tokens, targets, params, grad_targets=None):
        cfg = self.cfg
        if i == 0:  # embed: wte (shared) + wpe; with a target the wte gradient accumulates there (K13)
            wpe, wte = params
            T = tokens.shape[1]
            return _Embedding.apply(tokens, wte, grad_targets[0] if grad_targets else None) + wpe[:T]
        if i == self.K - 1:  # tied lm_head + loss (wte viewed with padded vocab rows)
            (wte,) = params
            # [B*T, vocab_padded] bf16 straight from the GEMM; with a target the wte gradient is written there
            logits = _TiedHead.apply(x.reshape(-1, x.shape[-1]), wte, cfg.vocab,
                                     grad_targets[0] if grad_targets else None)
            # K8: cross-entropy on the padded bf16 logits (pad columns excluded), gradient written
            # in place: no sliced fp32 copy of the 0.8 GB logits and no separate softmax kernels
            return kernels.lm_head_cross_entropy(logits.view(-1, logits.shape[-1]), targets.reshape(-1), cfg.vocab)
        if i == self.K - 2:  # ln_f
            w, b = params
            return layer_norm(x, w, b)
        return _block(x, params, cfg.heads, grad_targets)

    def pieces(self, i: int, lookup) -> list:
        """Node i's compute tensors cut from full parameters (lookup(pid))."""
        out = []
        for pid, off, shape in self.node_pieces[i]:
            t = lookup(pid)
            n = math.prod(shape)
            out.append(t if (off == 0 and n == t.numel()) else t.reshape(-1)[off:off + n].view(shape))
        return out

    def piece_grads_by_param(self, i: int, grads) -> dict:
        """Reassemble per-piece gradients into per-parameter gradients (tests)."""
        acc: dict[str, list] = {}
        for (pid, _, _), g in zip(self.node_pieces[i], grads):
            acc.setdefault(pid, []).append(g.reshape(-1))
        return {pid: torch.cat(gs).view(self.shapes[pid]) for pid, gs in acc.items()}

    def _params_of(self, i: int):
        ps = self.pieces(i, self.manager.param)
        if i == 0 or i == self.K - 1:
            self.optimizer.wait_gpu("wte", torch.cuda.current_stream(self.device))
            ps.append(self.manager.padded_param("wte", (self.cfg.vocab_padded, self.cfg.hidden)))
        return ps

    # -------------------------------------------------------------- step
    def train_step(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        """One chunked training step; returns the loss as a device scalar."""
        if tokens.device != self.device:
            raise ValidationError("tokens must already be on the trainer's device")
        fx, mgr = self.fetcher, self.manager
        K = self.K
        fx.inv_scale = 1.0 / self.scaler.scale
        fx.begin_step(after=self.optimizer.done_event)
        self.optimizer.wait_gpu("wte", torch.cuda.current_stream(self.device))
        acts = []
        saved = [None] * K
        x = None
        for i in range(K):
            fx.enter(i)
            acts.append(x)
            if i < K - 1 and self.keep_graph:  # keep the node's graph for the backward (no recompute)
                raw = self._params_of(i)
                params = [p.detach().requires_grad_(True) for p in raw]
                layer = 0 < i < K - 2
                xin = None if i == 0 else x.detach().requires_grad_(True)
                with torch.enable_grad():
                    out = self._run_node(i, xin, tokens, targets, params, grad_targets=self._targets(i, raw))
                saved[i] = (out, xin, params)
                x = out.detach()
            elif i < K - 1:  # the head's loss comes from its backward recompute
                with torch.no_grad():
                    x = self._run_node(i, x, tokens, targets, self._params_of(i))
            fx.after_compute(i)
        loss = None
        grad = torch.full((), self.scaler.scale, dtype=torch.float32, device=self.device)
        wte_grad_set = False
        for j in range(K):
            i = K - 1 - j
            pos = K + j
            fx.enter(pos)
            layer = 0 < i < K - 2
            if saved[i] is not None:
                out, xin, params = saved[i]
                saved[i] = None
            else:
                raw = self._params_of(i)
                params = [p.detach().requires_grad_(True) for p in raw]
                with torch.enable_grad():
                    xin = None if i == 0 else acts[i].detach().requires_grad_(True)
                    # layers: linear gradients land in their chunk slots (raw views) directly
                    out = self._run_node(i, xin, tokens, targets, params, grad_targets=self._targets(i, raw))
            with torch.enable_grad():
                inputs = ([xin] if i > 0 else []) + params
                grads = torch.autograd.grad(out, inputs, grad_outputs=grad, allow_unused=i != K - 2)
            if i == K - 1:
                loss = out.detach()
            acts[i] = None
            if i > 0:
                grad, pgrads = grads[0], grads[1:]
            else:
                pgrads = grads
            chunk_grads = pgrads[:len(self.node_pieces[i])]
            self._write_grads(i, chunk_grads)
            if (i == 0 or i == K - 1) and pgrads[-1] is None:  # written in place (_TiedHead, then K13)
                wte_grad_set = True
            elif i == 0 or i == K - 1:
                wg = pgrads[-1].reshape(-1)[:self.wte.numel]
                buf = self.wte.grad[:self.wte.numel]
                if wte_grad_set:
                    buf.add_(wg)
                else:
                    kernels.chunk_pack(self.wte.grad, [(wg, 0)], used_len=self.wte.numel)
                    wte_grad_set = True
            fx.after_compute(pos)
            del grads, pgrads, params, out
        fx.release_shared(self.wte)
        done = fx.finish()
        stats = self.optimizer.step(done, grad_scale=1.0 / self.scaler.scale)
        if self.scaler.dynamic:  # fp16: the next step's scale depends on this step's overflow (syncs)
            self.scaler.update(stats.found_inf)
        self.last_loss = loss
        return loss

    def _targets(self, i: int, raw):
        """Where node i's wrapped operators write their parameter gradients:
        a layer's chunk slots (aliases); for the tied head (first in the
        backward) and then the embedding, the shared wte gradient buffer."""
        if 0 < i < self.K - 2:
            return [_alias(t) for t in raw]
        if i == 0 or i == self.K - 1:
            return [self.wte.grad[:self.wte.numel].view(self.cfg.vocab, self.cfg.hidden)]
        return None

    def _write_grads(self, i: int, grads) -> None:
        """Overwrite the node's parameter slots in the chunk with their
        gradients (Fig. 3): one K1 launch per chunk."""
        by_chunk: dict[int, list] = {}
        for (pid, sub, _), g in zip(self.node_pieces[i], grads):
            if g is None:  # written in place by a wrapped operator (linear, LayerNorm)
                continue
            c, off, _ = self.manager.members[pid]
            by_chunk.setdefault(c, []).append((g.reshape(-1), off + sub))
        for c, mem in by_chunk.items():
            st = self.manager.storage(c)
            kernels.chunk_pack(st, mem, used_len=st.numel())

    def synchronize(self) -> None:
        """Make the current stream wait for every outstanding update (end of
        a timed region / before reading parameters)."""
        self.optimizer.synchronize()

    # -------------------------------------------------------------- CUDA graph
    def capture(self, tokens: torch.Tensor, targets: torch.Tensor, warmup: int = 3) -> None:
        """Capture one whole training step — forward, backward with the
        gradient write-backs, the K3 releases on the comm stream, the K4
        update and the device step counter — as ONE CUDA graph, so a step is a
        single graph launch instead of ~1400 host-issued kernels (the small
        GPT-2 step is launch-bound in eager mode). `warmup` eager steps run
        first (they train, like any step) on a side stream. The captured step
        depends on nothing outside the graph: every side stream rejoins the
        capture stream, and consecutive replays on one stream are ordered.
        Needs every chunk GPU-home (no host-thread update), a static loss
        scale, and world 1 or a graph-safe P2P transport (IpcTransport: every
        exchange is our kernels over peer memory, ordered by device-numbered
        barriers, so N ranks replay N graphs in lockstep without a collective
        library); the inputs of each later step are copied into the captured
        input buffers by graph_step()."""
        mgr = self.manager
        multi_ok = mgr.world == 1 or (mgr.p2p and getattr(mgr.transport, "graph_safe", False))
        if mgr.cpu_ids or self.scaler.dynamic or self.optimizer.overlap or not multi_ok:
            raise ValidationError("graph capture needs every chunk GPU-home, a static loss scale, the "
                                  "single-launch optimizer, and world 1 or a graph-safe P2P transport")
        self._g_tok = tokens.detach().clone()
        self._g_tgt = targets.detach().clone()
        if self.optimizer.tables is not None:
            self.optimizer.tables.ensure(1 << 20)  # the captured table pointers must stay valid
        cur = torch.cuda.current_stream(self.device)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self.train_step(self._g_tok, self._g_tgt)
            self.synchronize()
        cur.wait_stream(side)
        torch.cuda.synchronize(self.device)
        # nothing recorded before the capture may be waited on inside it
        self.optimizer.done_event = None
        self.optimizer.pending = {}
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            loss = self.train_step(self._g_tok, self._g_tgt)
            self.synchronize()
        self.optimizer.done_event = None  # events recorded during capture are graph-internal
        self._graph, self._g_loss = graph, loss

    def graph_step(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        """One training step by replaying the captured graph on new inputs
        (same shapes); returns the loss (a device scalar, overwritten by the
        next replay)."""
        if getattr(self, "_graph", None) is None:
            raise ValidationError("call capture() first")
        self._g_tok.copy_(tokens, non_blocking=True)
        self._g_tgt.copy_(targets, non_blocking=True)
        self._graph.replay()
        self.last_loss = self._g_loss
        return self._g_loss

    def release_graph(self) -> None:
        """Drop the captured step (its private memory pool: the kept
        activations and workspaces of one step) so an eager step can run in
        that memory; graph_step needs capture() again afterwards."""
        torch.cuda.synchronize(self.device)
        self._graph = self._g_loss = None
        self.last_loss = None if not isinstance(self.last_loss, torch.Tensor) else self.last_loss.clone()
        torch.cuda.empty_cache()

    # -------------------------------------------------------------- misc
    @property
    def n_params(self) -> int:
        return self.profile.total_elements

    def flops_per_step(self) -> float:
        """Executed model FLOPs for this rank's batch: 8·M·D with per-layer
        recompute (cost_model.py:170-174), 6·M·D when the
        forward graphs are kept."""
        return (6.0 if self.keep_graph else 8.0) * self.n_params * self.cfg.batch * self.cfg.seq_len
