"""Test infrastructure: a plain reference training step (standalone tensors,
same node functions, CPU oracle release + AdamW) and an in-process loopback
transport that runs N ranks as N threads on ONE GPU."""

from __future__ import annotations

import threading

import numpy as np
import torch

from oracle import arith


class ReferenceStep:
    """Standalone parameter tensors + the model's node functions + the CPU
    oracle optimizer. `step(batches)` takes one (tokens, targets) pair per
    rank; gradients of rank r are reduced in rank order exactly as the
    runtime's release does."""

    def __init__(self, model, init, hp):
        self.m = model
        self.hp = hp
        self.p16 = {k: v.clone() for k, v in init.items()}
        self.master = {k: v.float().cpu().numpy().reshape(-1).copy() for k, v in init.items()}
        self.mom = {k: np.zeros_like(v) for k, v in self.master.items()}
        self.vel = {k: np.zeros_like(v) for k, v in self.master.items()}
        self.t = 0

    def _grads(self, tokens, targets, scale):
        m = self.m
        K = m.K
        cfg = m.cfg
        wpad = torch.zeros(cfg.vocab_padded, cfg.hidden, dtype=self.p16["wte"].dtype, device=tokens.device)
        wpad[:cfg.vocab] = self.p16["wte"]

        def params(i):  # the same compute pieces (q/k/v row blocks) the runtime uses
            ps = m.pieces(i, self.p16.__getitem__)
            if i in (0, K - 1):
                ps.append(wpad)
            return ps

        acts, x = [], None
        with torch.no_grad():
            for i in range(K - 1):
                acts.append(x)
                x = m._run_node(i, x, tokens, targets, params(i))
        acts.append(x)
        grad = torch.full((), scale, dtype=torch.float32, device=tokens.device)
        grads, loss = {}, None
        for i in reversed(range(K)):
            raw = params(i)
            ps = [p.detach().requires_grad_(True) for p in raw]
            layer = 0 < i < K - 2
            # standalone gradient destinations for the wrapped linears (the runtime
            # writes into the chunk slots instead)
            tgt = [torch.empty_like(p) for p in raw] if layer else None
            with torch.enable_grad():
                xin = None if i == 0 else acts[i].detach().requires_grad_(True)
                out = m._run_node(i, xin, tokens, targets, ps, grad_targets=tgt)
                gs = torch.autograd.grad(out, ([xin] if i else []) + ps, grad_outputs=grad, allow_unused=layer)
            if i == K - 1:
                loss = out.detach()
            if i:
                grad, gs = gs[0], gs[1:]
            full = list(gs)
            pgs = full[:len(m.node_pieces[i])]
            if layer:
                pgs = [t if g is None else g for g, t in zip(pgs, tgt)]
            grads.update(m.piece_grads_by_param(i, pgs))
            if i in (0, K - 1):
                gw = full[-1][:cfg.vocab]
                grads["wte"] = gw if "wte" not in grads else grads["wte"] + gw
        return loss, grads

    def step(self, batches, scale=1.0):
        per_rank = [self._grads(tok, tgt, scale) for tok, tgt in batches]
        name = "bf16" if self.m.manager.dtype == torch.bfloat16 else "f16"
        rel, sq, bad = {}, 0.0, False
        for pid in per_rank[0][1]:
            srcs = [g[pid].detach().reshape(-1).cpu().view(torch.int16).numpy().view(np.uint16)
                    for _, g in per_rank]
            r, _, b = arith.release(srcs, 1.0 / scale, name)
            rel[pid], bad = r, bad or b
        # K3's sum-of-squares units run over each chunk from its offset 0 (oracle/arith.py quad_sq)
        sq = arith.sumsq_chunked(rel, self.m.manager.members)
        hp = self.hp
        coef = arith.clip_coef(sq, hp["max_norm"])
        t = self.t if bad else self.t + 1
        for pid in rel:
            p, mm, vv, p16 = arith.adamw(self.master[pid], self.mom[pid], self.vel[pid], rel[pid], max(t, 1),
                                         hp["lr"], hp["betas"][0], hp["betas"][1], hp["eps"], hp["weight_decay"],
                                         coef, bad, name)
            self.master[pid], self.mom[pid], self.vel[pid] = p, mm, vv
            t16 = torch.from_numpy(p16.view(np.int16)).view(self.p16[pid].dtype).view(self.p16[pid].shape)
            self.p16[pid] = t16.to(self.p16[pid].device)
        self.t = t
        return [l for l, _ in per_rank], bad


class LoopbackGroup:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world, timeout=120)
        self.slots = [None] * world


class LoopbackTransport:
    """N ranks = N threads sharing one GPU. Collectives exchange device
    tensors through a shared slot table with host barriers and stream syncs
    (slow, but exact: it moves bytes exactly as all_gather_into_tensor /
    all_to_all_single / all_reduce would)."""

    def __init__(self, group: LoopbackGroup, rank: int):
        self.g = group
        self.world = group.world
        self.rank = rank

    def _publish(self, t):
        torch.cuda.current_stream().synchronize()
        self.g.slots[self.rank] = t
        self.g.barrier.wait()
        return list(self.g.slots)

    def _done(self):
        torch.cuda.current_stream().synchronize()
        self.g.barrier.wait()

    def gather(self, block, shard):
        S = shard.numel()
        shards = self._publish(shard)
        for r, s in enumerate(shards):
            block[r * S:(r + 1) * S].copy_(s)
        self._done()

    def scatter(self, recv, block):
        S = recv.numel() // self.world
        blocks = self._publish(block)
        for r, b in enumerate(blocks):
            recv[r * S:(r + 1) * S].copy_(b[self.rank * S:(self.rank + 1) * S])
        self._done()

    def all_reduce_sum(self, t):
        ts = self._publish(t)
        acc = ts[0].clone()
        for x in ts[1:]:
            acc += x
        self._done()
        t.copy_(acc)
        self._done()

    def barrier(self):
        self.g.barrier.wait()


class LoopbackP2PTransport(LoopbackTransport):
    """Emulates the symmetric-memory path on one GPU: the 'peer pointers' are
    the other rank-threads' tensors on the same device, and the device barrier
    is a stream sync + host barrier (same ordering guarantee, blocking)."""

    p2p = True

    def alloc(self, shape, dtype, device):
        return torch.zeros(shape, dtype=dtype, device=device)

    def peer_ptrs(self, t):
        if t.numel() == 0:
            return [0] * self.world
        ts = self._publish(t)
        ptrs = [x.data_ptr() for x in ts]
        self._done()
        return ptrs

    def device_barrier(self):
        self._done()


def run_ranks(world: int, fn, p2p: bool = False):
    """Run fn(rank, transport) in `world` threads; re-raise the first error."""
    group = LoopbackGroup(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r, (LoopbackP2PTransport if p2p else LoopbackTransport)(group, r))
        except BaseException as exc:  # pragma: no cover - surfaced below
            errs.append(exc)
            group.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out
