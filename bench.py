"""Benchmark: chunked GPT-2 1.3B training step (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model gpt2-1.3b] [--sweep]

One process per GPU (torchrun for N > 1, NCCL). Each rank trains GPT-2 with
a per-rank micro-batch of 8 x 1024 synthetic tokens (weak scaling) through the
Elixir chunk runtime with the reference planner's plan for N GPUs
(plans/<model>_n<N>.json, made by offplan.build_plan). Prints ONE JSON line
(rank 0): samples/s (whole job), the chunk-Adam roofline, per-kernel rates,
the end-to-end rate through the public API with host buffers, the CPU
baseline, clocks and the number of our kernel launches.

--impl reference times the CPU path (oracle port: torch-CPU GPT-2 math + the
C oracle's release/AdamW) on host cores, on a bounded sample, scaled to
samples/s of the same workload.

--sweep runs the standalone K2/K3/K4 kernels over chunk sizes 4-256 MB
(BASELINE.json configs[4]) and prints one JSON line per size instead.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train step samples/sec (GPT-2 chunked, Elixir rCache) + chunk Adam HBM GB/s + fetch/RS bus GB/s"
# K4 algorithmic bytes per element: p32, m, v read + write (24) + gradient read (fp32 4, or the bf16
# gradient in place at world 1: 2) + bf16 parameter write (2) -> 30 or 28 (HybridAdam.bytes_per_element)


def _peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- distributed

def _dist_setup(n_gpus: int):
    """One process per GPU over NCCL. When fewer GPUs than ranks are visible
    (the one-GPU development box), the ranks share device `local % count` and
    talk over gloo — a functional run of the N>1 code path (sharding, rCache,
    all-gather / all-to-all + K3, the scalar all-reduce, max-over-ranks
    timing), flagged `oversubscribed` in the JSON line: not a scaling number."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    ndev = max(1, torch.cuda.device_count())
    shared = world > ndev
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    return world, rank, dev_index, (f"{world} ranks on {ndev} GPU(s) over gloo" if shared else None)


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


# ---------------------------------------------------------------- CPU baseline

def cpu_baseline(model_name: str, layers_sample: int = 2, threads: int | None = None, reps: int = 3):
    """Oracle-port CPU training step on a bounded sample, scaled to samples/s.

    Sample: ONE sequence (1024 tokens) through `layers_sample` transformer
    layers (forward + AC recompute + backward, torch CPU fp32) plus the tied
    lm_head/loss, and the C oracle's release + AdamW over those layers' chunk
    elements; the median of `reps` repetitions of each part (the host is
    shared: single samples spread by tens of percent). Scaled: per-layer time
    x L, optimizer time x (M / sampled elements), giving seconds per sequence
    of the full model.
    """
    import numpy as np
    from oracle.gpt2_ref import block as _block
    from paper_2212_05339_b200.gpt2 import PRESETS
    import torch.nn.functional as F

    cfg = PRESETS[model_name]
    cores = len(os.sched_getaffinity(0))
    threads = threads or cores
    torch.set_num_threads(threads)
    h, T, V = cfg.hidden, cfg.seq_len, cfg.vocab
    g = torch.Generator().manual_seed(0)
    layer_params = [
        [torch.ones(h), torch.zeros(h)] + [torch.randn(h, h, generator=g) * 0.02 for _ in range(3)]
        + [torch.zeros(h) for _ in range(3)] + [
         torch.randn(h, h, generator=g) * 0.02, torch.zeros(h), torch.ones(h), torch.zeros(h),
         torch.randn(4 * h, h, generator=g) * 0.02, torch.zeros(4 * h), torch.randn(h, 4 * h, generator=g) * 0.02,
         torch.zeros(h)] for _ in range(layers_sample)]
    wte = torch.randn(V, h, generator=g) * 0.02
    x0 = torch.randn(1, T, h, generator=g)
    tgt = torch.randint(0, V, (1, T), generator=g)

    def layer_pass(ps, x):
        with torch.no_grad():
            _block(x, ps, cfg.heads)
        q = [p.clone().requires_grad_(True) for p in ps]
        xi = x.clone().requires_grad_(True)
        out = _block(xi, q, cfg.heads)
        gr = torch.autograd.grad(out, [xi] + q, torch.ones_like(out))
        return gr[0]

    def layers_once():
        t0 = time.perf_counter()
        for ps in layer_params:
            layer_pass(ps, x0)
        return (time.perf_counter() - t0) / layers_sample

    def head_once():
        t0 = time.perf_counter()
        w = wte.clone().requires_grad_(True)
        xi = x0.clone().requires_grad_(True)
        with torch.no_grad():
            F.cross_entropy(F.linear(x0, wte).view(-1, V), tgt.view(-1))
        loss = F.cross_entropy(F.linear(xi, w).view(-1, V), tgt.view(-1))
        torch.autograd.grad(loss, [xi, w])
        return time.perf_counter() - t0

    t_layers = statistics.median(layers_once() for _ in range(reps))
    t_head = statistics.median(head_once() for _ in range(reps))

    # optimizer: C oracle release (world 1) + AdamW over the sampled layers' elements
    lib = ctypes.CDLL(str(ROOT / "oracle" / "_build" / "liboracle.so"))
    lib.oracle_release_bf16.restype = ctypes.c_double
    lib.oracle_release_bf16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int]
    lib.oracle_adamw_bf16.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                                             ctypes.c_int, ctypes.c_int]
    n = layers_sample * (12 * h * h + 13 * h)
    gb = np.zeros(n, np.uint16)
    p = np.full(n, 0.01, np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    g32 = np.zeros(n, np.float32)
    p16 = np.zeros(n, np.uint16)
    ptrs = (ctypes.c_void_p * 1)(gb.ctypes.data)
    bad = ctypes.c_int(0)
    k = np.array([1 - 1e-5, 0.1, 0.999, 0.001, 0.0316, -0.01, 1e-8], np.float32)
    def opt_once():
        t0 = time.perf_counter()
        lib.oracle_release_bf16(g32.ctypes.data, ptrs, 1, n, ctypes.c_float(1.0), ctypes.byref(bad), threads)
        lib.oracle_adamw_bf16(p.ctypes.data, m.ctypes.data, v.ctypes.data, g32.ctypes.data, p16.ctypes.data, n,
                              k.ctypes.data, ctypes.c_float(1.0), 0, threads)
        return time.perf_counter() - t0

    t_opt = statistics.median(opt_once() for _ in range(reps))
    total = 12 * h * h * cfg.layers + 13 * h * cfg.layers + V * h + T * h + 2 * h
    sec_per_seq = t_head + cfg.layers * t_layers + t_opt * total / n
    return {
        "value": 1.0 / sec_per_seq,
        "unit": "samples/s",
        "cores": threads,
        "kind": "port",
        "sample": (f"1 sequence x {T} tokens through {layers_sample} of {cfg.layers} layers + tied lm_head "
                   f"(torch CPU fp32, fwd+recompute+bwd) and C-oracle release+AdamW over {n} elements, median of "
                   f"{reps} repetitions each; scaled to the full {total}-parameter model"),
        "seconds_measured": round(reps * (t_layers * layers_sample + t_head + t_opt), 3),
        "breakdown_s_per_seq": {"layers": cfg.layers * t_layers, "head": t_head, "optimizer": t_opt * total / n},
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(args.model, reps=1)  # one sample per step: the median is over the steps
        if i >= args.warmup:
            vals.append(cb["value"])
    value = statistics.median(vals)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.model} chunked training step (CPU oracle port)", "model": args.model,
                   "seq_len": 1024, "per_rank_batch": 8},
        "cpu_baseline": {**{k: cb[k] for k in ("kind", "cores", "sample")}, "value": value, "unit": "samples/s"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------- GPU arm

def _fetch_stats(fet, world, steps, kind):
    """K2 (or the library all-gather) per gather: (ms, block elements) pairs
    from the eager probe steps; busBW = (N-1)/N * 2 B * P / t (NCCL's busBw
    convention for an all-gather of P elements)."""
    engine = {"ipc": "K2 on SMs reading peers' shards through our CUDA-IPC mappings (NVLink)",
              "ipc-ce": "K2 on the copy engines (cudaMemcpyAsync per peer) over CUDA-IPC mappings",
              "p2p": "K2 on SMs reading peers' shards through torch symmetric memory",
              "nccl": "NCCL all_gather_into_tensor on the comm stream"}.get(kind, kind)
    if not fet:
        return {"engine": engine, "gathers_timed": 0}
    ms = sum(t for t, _ in fet)
    nbytes = sum((world - 1) / world * 2 * n for _, n in fet)
    return {"engine": engine, "gathers_per_step": len(fet) / max(1, steps), "ms_per_step": ms / max(1, steps),
            "ms_per_gather": ms / len(fet), "bus_gbs": nbytes / (ms * 1e-3) / 1e9,
            "bus_frac_of_900": nbytes / (ms * 1e-3) / 1e9 / 900,
            "note": "CUDA events around each gather on the comm stream (eager probe steps when the step is a graph)"}


def _release_alone(model, dev, cur):
    from paper_2212_05339_b200 import kernels
    mgr = model.manager
    scratch = kernels.new_step_scalars(dev)
    fx = model.fetcher
    todo = [(None, [mgr.home_storage(c).data_ptr()], mgr.valid(c)) for c in mgr.gpu_ids if mgr.valid(c) > 0]
    groups = [[(None, [mgr.home_storage(c).data_ptr()], mgr.valid(c)) for c in fx.reduces[p]
               if mgr.homes[c].value == "gpu" and mgr.valid(c) > 0] for p in range(len(fx.reduces))]
    groups = [g for g in groups if g]
    n_alone = sum(n for _, _, n in todo)
    peak = _peaks()[0]

    def timed(fn, reps=10):
        ts = []
        for i in range(reps + 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            fn()
            b.record(cur)
            torch.cuda.synchronize(dev)
            if i >= 3:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    ms_batch = timed(lambda: kernels.release_batch(todo, mgr.dtype, 1.0, scratch, stream=cur))
    side = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        for grp in groups:  # warm the launch path outside the capture
            kernels.release_batch(grp, mgr.dtype, 1.0, scratch, stream=side)
    cur.wait_stream(side)
    torch.cuda.synchronize(dev)
    with torch.cuda.graph(g):
        for grp in groups:
            kernels.release_batch(grp, mgr.dtype, 1.0, scratch)
    ms_graph = timed(g.replay)
    gbs = lambda ms: 2 * n_alone / (ms * 1e-3) / 1e9
    return {"elements": n_alone, "bytes_per_element": 2,
            "batched": {"ms": ms_batch, "launches": 1, "hbm_gbs": gbs(ms_batch), "frac": gbs(ms_batch) / peak},
            "per_reduce_position": {"ms": ms_graph, "launches": len(groups), "hbm_gbs": gbs(ms_graph),
                                    "frac": gbs(ms_graph) / peak, "note": "the step's launch pattern, CUDA graph"},
            "ms": ms_batch, "hbm_gbs": gbs(ms_batch), "frac": gbs(ms_batch) / peak}


def run_ours(args):
    from paper_2212_05339_b200 import _lib
    from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2

    world, rank, local, oversub = _dist_setup(args.gpus)
    if oversub and args.transport == "p2p":
        raise SystemExit("--transport p2p needs one GPU per rank (symmetric memory refuses a shared device)")
    dev = torch.device("cuda", local)
    cfg = PRESETS[args.model]
    if args.batch:
        import dataclasses
        cfg = dataclasses.replace(cfg, batch=args.batch)
    plan_path = ROOT / "plans" / (args.plan.format(n=world) if args.plan else f"{args.model}_n{world}.json")
    plan_text = plan_path.read_text()
    from paper_2212_05339_b200.transport import make_transport, primary_contexts, resolve_kind
    kind = resolve_kind(world, args.transport)
    transport = make_transport(world, kind)
    model = ElixirGPT2(cfg, plan_text, device=dev, seed=1234, transport=transport,
                       overlap_update=args.overlap, cpu_update=args.cpu_update,
                       recompute={"auto": "auto", "on": True, "off": False}[args.recompute])
    B, T = cfg.batch, cfg.seq_len
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    ids = torch.randint(0, cfg.vocab, (B, T + 1), generator=gen, device=dev)
    tok, tgt = ids[:, :-1].contiguous(), ids[:, 1:].contiguous()

    for _ in range(args.warmup):
        model.train_step(tok, tgt)
    _barrier(world)

    opt = model.optimizer
    cur = torch.cuda.current_stream(dev)

    def timing(on: bool) -> None:
        opt.time_adam = on
        model.fetcher.time_release = on
        if on:
            opt.adam_events.clear()
            model.fetcher.release_events.clear()
            model.fetcher.fetch_events.clear()
            model.fetcher.copy_events.clear()
            opt.cpu_wait_s = opt.cpu_update_s = 0.0
            opt.stream_events.clear()

    # CUDA graph: the whole step as one graph launch (every chunk GPU-home; world 1, or N ranks on the
    # IPC P2P transport, whose exchanges are our kernels between device-numbered barriers). The per-kernel
    # event timings then come from `warmup` eager steps of the same launches, run just before capture.
    use_graph = (args.graph and not model.manager.cpu_ids and
                 (world == 1 or (model.manager.p2p and getattr(model.manager.transport, "graph_safe", False))))
    step_fn = model.train_step
    probe_steps = args.steps
    if use_graph:
        timing(True)
        l0 = _lib.launch_count()
        for _ in range(args.warmup):
            model.train_step(tok, tgt)
        model.synchronize()
        torch.cuda.synchronize(dev)
        per_step_launches = (_lib.launch_count() - l0) / args.warmup
        probe_steps = args.warmup
        timing(False)
        # K4 timed INSIDE the captured step: event-record nodes around it, re-recorded by every replay
        k4_graph_events = opt.prepare_graph_timing()
        opt.time_adam = True
        model.capture(tok, tgt, warmup=1)
        opt.time_adam = False
        opt.adam_events.clear()
        step_fn = model.graph_step
    else:
        timing(True)

    # ---- device-resident timed region
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        _barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(args.steps):
            step_fn(tok, tgt)
        model.synchronize()  # the last step's overlapped update is inside the timed region
        e1.record(cur)
        torch.cuda.synchronize(dev)
    launches = _lib.launch_count() - l0
    k4_in_graph = None
    if use_graph:  # our kernels run inside the graph replays: the captured step's launches, per replay
        launches = int(round(per_step_launches * args.steps))
        # the last timed replay's K4, then a few more replays read one by one (graph-internal events)
        e_a, e_b = k4_graph_events
        k4_in_graph = [e_a.elapsed_time(e_b)]
        for _ in range(4):
            step_fn(tok, tgt)
            torch.cuda.synchronize(dev)
            k4_in_graph.append(e_a.elapsed_time(e_b))
    ms = e0.elapsed_time(e1)
    ms = _max_over_ranks(ms, world)
    adam_ms = [a.elapsed_time(b) for a, b in opt.adam_events]
    rel = [(a.elapsed_time(b), n) for a, b, n in model.fetcher.release_events]
    fet = [(a.elapsed_time(b), n) for a, b, n in model.fetcher.fetch_events]
    copies = {}
    for ckind, a, b, nb in model.fetcher.copy_events:
        ms_, nb0 = copies.get(ckind, (0.0, 0))
        copies[ckind] = (ms_ + a.elapsed_time(b), nb0 + nb)
    cpu_wait_ms = opt.cpu_wait_s * 1e3 / probe_steps
    cpu_update_ms = opt.cpu_update_s * 1e3 / probe_steps
    stream_update_ms = (statistics.mean(a.elapsed_time(b) for a, b in opt.stream_events)
                        if opt.stream_events else 0.0)
    timing(False)
    loss = float(model.last_loss)

    # ---- end to end through the public API with host buffers
    host_ids = torch.randint(0, cfg.vocab, (B, T + 1), generator=torch.Generator().manual_seed(99 + rank)).pin_memory()
    dev_ids = torch.empty_like(host_ids, device=dev)
    loss_host = torch.zeros(2, dtype=torch.float32).pin_memory()   # one slot per step in flight
    e2e_losses = []
    _barrier(world)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(cur)
    # a non-blocking training loop: step i's tokens go up and its loss comes back on the compute stream;
    # the host reads step i's loss once step i+1 is enqueued (one step in flight), so the GPU never idles
    # on the host's wake-up and the next launch
    pending = None
    step_marks = []   # (start, done) per step: device time of the step vs the gaps between steps
    for i in range(args.steps):
        start = torch.cuda.Event(enable_timing=True)
        start.record(cur)
        dev_ids.copy_(host_ids, non_blocking=True)
        lo = step_fn(dev_ids[:, :-1], dev_ids[:, 1:])
        loss_host[i % 2].copy_(lo.reshape(()), non_blocking=True)
        done = torch.cuda.Event(enable_timing=True)
        done.record(cur)
        step_marks.append((start, done))
        if pending is not None:
            pending[0].synchronize()
            e2e_losses.append(float(loss_host[pending[1]]))
        pending = (done, i % 2)
    pending[0].synchronize()
    e2e_losses.append(float(loss_host[pending[1]]))
    model.synchronize()
    f1.record(cur)
    torch.cuda.synchronize(dev)
    e2e_ms = _max_over_ranks(f0.elapsed_time(f1), world)
    e2e_step_ms = statistics.median(a.elapsed_time(b) for a, b in step_marks)
    e2e_gap_ms = (statistics.median(step_marks[i][1].elapsed_time(step_marks[i + 1][0])
                                    for i in range(len(step_marks) - 1)) if len(step_marks) > 1 else 0.0)

    # ---- the same step with the reference's per-layer checkpointing (world 1, graph mode): the model keeps
    # training, its step is re-captured with the recompute on and timed the same way (reported beside the
    # headline, which keeps the forward graphs)
    checkpointed = None
    if world == 1 and use_graph and model.keep_graph:
        model.keep_graph = False
        model.capture(tok, tgt, warmup=1)
        torch.cuda.synchronize(dev)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(cur)
        for _ in range(args.steps):
            model.graph_step(tok, tgt)
        model.synchronize()
        c1.record(cur)
        torch.cuda.synchronize(dev)
        cms = c0.elapsed_time(c1)
        checkpointed = {"value": B * args.steps / (cms * 1e-3), "unit": "samples/s", "ms_per_step": cms / args.steps,
                        "note": "same model and plan, per-layer activation checkpointing (recompute in the backward), "
                                "CUDA graph, timed right after the headline"}
        model.keep_graph = True
        model._graph = None  # the captured graph is the checkpointed step: a later graph_step must re-capture

    # ---- K3 alone on the step's own chunks (world 1: the norm/overflow pass over every GPU-home
    # chunk, with the GPU otherwise idle): (a) the whole set as ONE batched launch (the kernel's own
    # rate), (b) the step's launch pattern — one launch per reduce position — replayed from a CUDA
    # graph, so host launch overhead is not in the number. In-step the releases run on the comm stream
    # concurrently with the backward's GEMMs, which stretches them.
    rel_alone = None
    if world == 1 and model.manager.gpu_ids:
        rel_alone = _release_alone(model, dev, cur)

    # ---- parity (the checker, after every timed region): one more eager step of the SAME model on the same
    # batch, its K3 launches logged and the K4 inputs snapshotted on the device; the C oracle recomputes the
    # sum of squares in each launch's fixed order and AdamW over every element (oracle/parity.py)
    # (N > 1: every rank checks its own shards, oracle/parity.check_step_multirank, merged on every rank)
    parity = None
    if not args.no_parity:
        if use_graph:
            model.release_graph()   # the eager checked step runs in the captured step's memory (N ranks per GPU)
        t0 = time.perf_counter()
        if world == 1:
            from oracle.parity import check_step
            parity = check_step(model, tok, tgt)
        else:
            from oracle.parity import check_step_multirank
            parity = check_step_multirank(model, tok, tgt)
        parity["seconds"] = round(time.perf_counter() - t0, 1)

    if rank != 0:
        return
    peak, peak_src = _peaks()
    adam_elems = opt.gpu_elements
    bpe = opt.bytes_per_element
    adam_probe = statistics.mean(adam_ms) if adam_ms else float("nan")
    # the roofline's K4 time: inside the timed CUDA-graph replays when the step is a graph, else the timed
    # eager steps' own K4 events
    adam_avg = statistics.median(k4_in_graph) if k4_in_graph else adam_probe
    adam_gbs = bpe * adam_elems / (adam_avg * 1e-3) / 1e9
    rel_ms = sum(r for r, _ in rel) / max(1, probe_steps)
    rel_elems = sum(n for _, n in rel) / max(1, probe_steps)
    es = 2  # bf16
    rel_local_bytes = rel_elems * (es * world + (0 if world == 1 else 4))  # world 1: norm/overflow pass only
    traffic = None
    tp = ROOT / "profiles" / "adam_ncu_traffic.json"
    if tp.exists():
        try:
            t = json.loads(tp.read_text())
            if t.get("valid_elements") == adam_elems and t.get("bytes_per_element", 30) == bpe:
                traffic = t["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    samples = world * B * args.steps
    value = samples / (ms * 1e-3)
    cpu = cpu_baseline(args.model) if (world == 1 and not args.no_cpu) else None
    homes = model.manager.homes
    offload = {"cpu_home_chunks": len(model.manager.cpu_ids), "gpu_home_chunks": len(model.manager.gpu_ids),
               "bytes_moved_per_step": {k: v for k, v in model.fetcher.bytes_moved.items()},
               "sim_counters": model.fetcher.counters(),
               "offload_copies_per_step": {k: {"ms": v[0] / probe_steps, "bytes": v[1] / probe_steps,
                                               "gbs": v[1] / (v[0] * 1e-3) / 1e9 if v[0] else None}
                                           for k, v in copies.items()},
               "cpu_update_ms_per_step": cpu_update_ms, "host_wait_on_cpu_update_ms_per_step": cpu_wait_ms,
               "stream_update_ms_per_step": stream_update_ms,
               "cpu_update_mode": args.cpu_update,
               "host_updated_chunks": sorted(opt.cpu_segs), "stream_updated_chunks": sorted(opt.stream_segs)}
    flops = model.flops_per_step()
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (uniform tokens, N(0,0.02) init, seed 1234+rank)",
        "config": {
            "workload": f"{args.model} chunked training step, plan {plan_path.name} (offplan.build_plan)",
            "model": args.model, "global_batch": world * B, "per_rank_batch": B, "seq_len": T,
            "parallelism": f"elixir-chunk-dp{world}", "transport": kind, "chunk_length": model.layout.chunk_length,
            "cuda_contexts_on_devices": primary_contexts(),
            "n_chunks": model.layout.n_chunks, "n_block": model.manager.plan.n_block,
            "l2": "working set (>20 GB of chunk/optimizer state per step) far exceeds the 126 MB L2; no flush needed",
            "cuda_graph": use_graph,
            "deterministic": bool(args.deterministic),
            "activation_checkpointing": not model.keep_graph,
            "recompute_note": ("off: every chunk stays resident forward->backward and the activations fit, so "
                               "each node's forward graph is kept instead of recomputed — results bit-identical "
                               "to checkpointing (tests/test_runtime_gpu.py::test_keep_graph_step_equals_"
                               "recompute); --recompute on for the reference's per-layer checkpointing"
                               if model.keep_graph else
                               "on: per-layer activation checkpointing (PAPER.md:145-150)"),
            **({"oversubscribed": oversub} if oversub else {}),
        },
        "tflops_per_gpu": flops / (ms / args.steps * 1e-3) / 1e12,
        "tflops_note": "executed model FLOPs: 6·M·D, plus 2·M·D for the recompute when checkpointing "
                       "(PAPER.md:356 counts 8·M·D)",
        "final_loss": loss,
        "kernels": {
            "chunk_adam": {"ms_per_launch": adam_avg, "valid_elements": adam_elems, "hbm_gbs": adam_gbs,
                           "launches_timed": len(k4_in_graph) if k4_in_graph else len(adam_ms),
                           "in_graph_ms": k4_in_graph,
                           "eager_probe_ms": adam_probe if use_graph else None,
                           "overlapped_with_next_forward": args.overlap,
                           "note": "per step: all K4 launches (one per chunk group) on the optimizer stream, "
                                   "timed first-to-last with CUDA events on that stream"
                                   + (": event-record nodes inside the captured step, read after the last timed "
                                      "replay and 4 more replays (median)" if use_graph else "")},
            "release": {"ms_per_step": rel_ms, "elements_per_step": rel_elems,
                        "local_hbm_gbs": rel_local_bytes / (rel_ms * 1e-3) / 1e9 if rel_ms else None,
                        "bus_gbs": (None if world == 1 else
                                    (world - 1) / world * 2 * rel_elems * world / (rel_ms * 1e-3) / 1e9),
                        "bus_frac_of_900": (None if world == 1 else
                                            (world - 1) / world * 2 * rel_elems * world / (rel_ms * 1e-3) / 1e9 / 900),
                        "bus_note": "busBW = (N-1)/N * 2 B * N * S / t per K3 launch (timed after its device barrier)",
                        "in_step_note": "comm stream, concurrent with the backward's GEMMs",
                        "alone": rel_alone},
            "fetch": ({"note": "N=1: GPU-home chunk shards are used in place (zero-copy gathers)"} if world == 1 else
                      _fetch_stats(fet, world, probe_steps, kind)),
        },
        "roofline": {"bound": "hbm", "kernel": "elx_adam (K4)", "achieved": adam_gbs, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": adam_gbs / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": bpe * adam_elems, "bytes_per_element": bpe,
                     # also against the nominal HBM3e rate (HGX B200, B200_PROFILING.md)
                     "nominal_peak": 7700.0, "frac_of_nominal": adam_gbs / 7700.0},
        "e2e": {"value": samples / (e2e_ms * 1e-3), "unit": "samples/s",
                "h2d_bytes_per_step": host_ids.numel() * host_ids.element_size(),
                "d2h_bytes_per_step": loss_host.element_size(),
                "api": ("ElixirGPT2.graph_step (the captured train_step)" if use_graph else "ElixirGPT2.train_step")
                       + " on tokens copied from pinned host memory every step, every step's loss read back "
                         "on the host (one step in flight)",
                "losses_read": len(e2e_losses), "all_finite": all(math.isfinite(x) for x in e2e_losses),
                "device_ms_per_step": e2e_step_ms, "gap_ms_between_steps": e2e_gap_ms},
        "checkpointed": checkpointed,
        "parity": parity,
        "chunk_runtime": offload,
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))


# ---------------------------------------------------------------- kernel sweep

def _sweep_parity_peers(mb, world, rank, S, block, pb, sc, dev, bar):
    """--sweep-check at N > 1 (real peer pointers): after the timed launches
    every rank's block holds the gathered shards (K2 last wrote them). Each
    rank regenerates every rank's shard from its seed and checks (a) its block's
    bytes == their concatenation, (b) K3 over segment `rank` of every peer's
    block — fresh step scalars, scale 1/8 — against the C oracle: the fp32
    reduction bit for bit and the sum of squares in the launch's order. Merged
    over ranks (every rank runs it; rank 0 prints)."""
    import ctypes

    import numpy as np
    import torch.distributed as dist

    from oracle import parity
    from paper_2212_05339_b200 import kernels

    lib = parity._lib()
    lib.oracle_release_bf16.restype = ctypes.c_double
    lib.oracle_release_bf16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int]
    lib.oracle_release_norm_ordered.restype = ctypes.c_double
    lib.oracle_release_norm_ordered.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int]
    threads = max(1, len(os.sched_getaffinity(0)) // world)
    shards = []
    for r in range(world):  # the shards exactly as run_sweep made them (seed 77 + r, first draw)
        g = torch.Generator(device=dev).manual_seed(77 + r)
        shards.append(torch.randn(S, generator=g, device=dev).to(torch.bfloat16).view(torch.int16).cpu()
                      .numpy().view(np.uint16))
    torch.cuda.synchronize(dev)
    k2 = bool(np.array_equal(block.view(torch.int16).cpu().numpy().view(np.uint16), np.concatenate(shards)))
    bar()
    g32 = torch.empty(S, device=dev)
    sc.zero_()
    kernels.release(g32, [p + rank * S * 2 for p in pb], S, torch.bfloat16, 0.125, sc)
    bar()  # peers' blocks are read before anyone moves on
    torch.cuda.synchronize(dev)
    mine = shards[rank]   # segment `rank` of every rank's block is this rank's shard
    ptrs = (ctypes.c_void_p * world)(*([mine.ctypes.data] * world))
    want = np.empty(S, np.float32)
    bad = ctypes.c_int(0)
    lib.oracle_release_bf16(want.ctypes.data, ptrs, world, S, ctypes.c_float(0.125), ctypes.byref(bad), threads)
    k3_g = bool(np.array_equal(g32.cpu().numpy().view(np.uint32), want.view(np.uint32)))
    ctas, tv = kernels.release_geometry([S], world)
    gp = (ctypes.c_void_p * 1)(want.ctypes.data)
    nn = (ctypes.c_int64 * 1)(S)
    k3_sq = float(sc[0].item()) == lib.oracle_release_norm_ordered(gp, nn, 1, ctas, tv, threads)
    allr = [None] * world
    dist.all_gather_object(allr, (k2, k3_g, k3_sq))
    return {"chunk_mb": mb, "engine": "parity", "shard_elems": S, "ranks": world,
            "k2_bytes_identical": all(a for a, _, _ in allr), "k3_grad_bit_identical": all(b for _, b, _ in allr),
            "k3_sumsq_bit_identical": all(c for _, _, c in allr), "oracle": "oracle/c/elx_oracle.c"}


def _sweep_parity(mb, w, S, shards, block, dev, hp):
    """--sweep-check: the sweep's kernels at this chunk size against the C
    oracle (the checker, after the timed launches): K2's gathered bytes; K3's
    rank-ordered fp32 reduction (N > 1) and its sum of squares in the launch's
    fixed order; K4 over one rank's shard from fresh state."""
    import ctypes

    import numpy as np

    from oracle import arith, parity
    from paper_2212_05339_b200 import kernels

    lib = parity._lib()
    lib.oracle_release_bf16.restype = ctypes.c_double
    lib.oracle_release_bf16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int]
    lib.oracle_release_norm_ordered.restype = ctypes.c_double
    lib.oracle_release_norm_ordered.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int]
    threads = len(os.sched_getaffinity(0))
    hp = dict(hp, max_norm=1.0)   # with clipping: K4 reads the sum of squares K3 left in the step scalars
    t0 = time.perf_counter()
    hs = [t.view(torch.int16).cpu().numpy().view(np.uint16) for t in shards]
    kernels.fetch(block, [t.data_ptr() for t in shards], S)
    torch.cuda.synchronize(dev)
    k2 = bool(np.array_equal(block.view(torch.int16).cpu().numpy().view(np.uint16), np.concatenate(hs)))
    # K3: release into a fresh fp32 shard and fresh step scalars, scale 1/8
    g32 = torch.empty(S, device=dev)
    sc = kernels.new_step_scalars(dev)
    kernels.release(g32, [t.data_ptr() for t in shards], S, torch.bfloat16, 0.125, sc)
    torch.cuda.synchronize(dev)
    want = np.empty(S, np.float32)
    bad = ctypes.c_int(0)
    ptrs = (ctypes.c_void_p * w)(*[h.ctypes.data for h in hs])
    lib.oracle_release_bf16(want.ctypes.data, ptrs, w, S, ctypes.c_float(0.125), ctypes.byref(bad), threads)
    k3_g = bool(np.array_equal(g32.cpu().numpy().view(np.uint32), want.view(np.uint32)))
    ctas, tv = kernels.release_geometry([S], w)
    gp = (ctypes.c_void_p * 1)(want.ctypes.data)
    nn = (ctypes.c_int64 * 1)(S)
    sq = lib.oracle_release_norm_ordered(gp, nn, 1, ctas, tv, threads)
    k3_sq = float(sc[0].item()) == sq
    # K4 from fresh state on the released gradient
    gen = torch.Generator(device=dev).manual_seed(mb * 10 + w)
    p32 = torch.randn(S, device=dev, generator=gen) * 0.02
    m = torch.randn(S, device=dev, generator=gen) * 1e-3
    v = torch.rand(S, device=dev, generator=gen) * 1e-6
    P, M, V = (t.cpu().numpy() for t in (p32, m, v))
    p16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
    tab = kernels.AdamTable([(p32, m, v, g32, p16, S)], dev)
    kernels.adam(tab, hp, 1, sc, torch.bfloat16)
    torch.cuda.synchronize(dev)
    coef = arith.clip_coef(sq, hp["max_norm"])
    k = arith.adam_consts(1, hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"])
    kv = np.array([k["decay"], k["omb1"], k["b2"], k["omb2"], k["bc2_sqrt"], k["neg_step"], k["eps"]], np.float32)
    out16 = np.empty(S, np.uint16)
    lib.oracle_adamw_bf16(P.ctypes.data, M.ctypes.data, V.ctypes.data, want.ctypes.data, out16.ctypes.data, S,
                          kv.ctypes.data, ctypes.c_float(coef), 0, threads)
    k4 = all(np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32)) for a, b in ((p32, P), (m, M), (v, V)))
    k4 = k4 and bool(np.array_equal(p16.view(torch.int16).cpu().numpy().view(np.uint16), out16))
    return {"chunk_mb": mb, "emulated_world": w, "engine": "parity", "shard_elems": S,
            "k2_bytes_identical": k2, "k3_grad_bit_identical": k3_g, "k3_sumsq_bit_identical": k3_sq,
            "k4_bit_identical": bool(k4), "oracle": "oracle/c/elx_oracle.c", "seconds": round(time.perf_counter() - t0, 1)}


def _sweep_graph_stream(mb, w, S, dev, reps, flush, flush_sink, hp, peak, emit):
    """The sweep's kernels as the step issues them: R back-to-back launches,
    each on its OWN buffers (R x the per-launch bytes >= 512 MB, four times
    the L2, so no launch reads what an earlier one left in L2), captured as
    one CUDA graph and replayed; ms per launch = replay time / R. A single
    cold launch of a few-MB chunk is dominated by launch latency and the DRAM
    ramp (the plain sweep lines); this is the per-chunk cost inside a step."""
    from paper_2212_05339_b200 import kernels

    sc = kernels.new_step_scalars(dev)
    engines = {
        "k2_fetch_sm": 2 * 2 * w * S,
        "k2_fetch_ce": 2 * 2 * w * S,
        "k3_release": 2 * w * S + (4 * S if w > 1 else 0),
        "k4_adam": 30 * S,
    }
    for engine, nbytes in engines.items():
        R = max(1, min(64, -(-(512 * 2 ** 20) // nbytes)))
        launches = []
        for _ in range(R):
            if engine.startswith("k2"):
                shards = [torch.randn(S, device=dev).to(torch.bfloat16) for _ in range(w)]
                block = torch.empty(w * S, dtype=torch.bfloat16, device=dev)
                ce = "ce" if engine.endswith("ce") else "sm"
                launches.append((lambda b=block, ps=[t.data_ptr() for t in shards], e=ce:
                                 kernels.fetch(b, ps, S, engine=e), (shards, block)))
            elif engine == "k3_release":
                shards = [torch.randn(S, device=dev).to(torch.bfloat16) for _ in range(w)]
                g32 = torch.empty(S, device=dev) if w > 1 else None
                launches.append((lambda g=g32, ps=[t.data_ptr() for t in shards]:
                                 kernels.release(g, ps, S, torch.bfloat16, 1.0, sc), (shards, g32)))
            else:
                p32, m, v = (torch.zeros(S, device=dev) for _ in range(3))
                g32 = torch.randn(S, device=dev)
                p16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
                tab = kernels.AdamTable([(p32, m, v, g32, p16, S)], dev)
                launches.append((lambda t=tab: kernels.adam(t, hp, 1, sc, torch.bfloat16), (p32, m, v, g32, p16)))
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for f, _ in launches:
                f()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for f, _ in launches:
                f()
        ts = []
        for i in range(reps + 2):
            torch.sum(flush, dim=0, out=flush_sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graph.replay()
            b.record()
            torch.cuda.synchronize(dev)
            if i >= 2:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts) / R
        emit({"chunk_mb": mb, "emulated_world": w, "engine": engine, "shard_elems": S, "mode": "graph_stream",
              "launches_per_graph": R, "ms": ms, "hbm_gbs": nbytes / (ms * 1e-3) / 1e9,
              "frac": nbytes / (ms * 1e-3) / 1e9 / peak})
        del graph, launches
        torch.cuda.empty_cache()


def run_sweep(args):
    """configs[4]: the chunk sweep — K2 fetch (SMs and copy engines), K3
    release and K4 Adam over chunk sizes 4-256 MB, at N = WORLD_SIZE ranks.

    N > 1 (torchrun, one process per GPU): every rank allocates its shard of a
    chunk and an rCache block, peers map each other's buffers (our CUDA-IPC
    mappings, or torch symmetric memory with --transport p2p), and each engine
    runs on REAL peer pointers between device barriers: K2 reads the N shards
    into the block (all-gather), K3 reduces segment `rank` of every peer's
    block (reduce-scatter + unscale + norm). NCCL's all_gather_into_tensor and
    reduce_scatter_tensor (bf16 and fp32) run on the same buffers as the bar.
    busBW = (N-1)/N * bytes / t (NCCL's convention; bytes = the gathered block
    or the reduce-scatter input), against 900 GB/s per direction. Time = max
    over ranks of the median of `reps` launches, each started after a device
    barrier, L2 flushed by a 256 MB read before each. Ranks sharing one GPU
    (the one-GPU box) run the same code as a functional check, flagged
    `oversubscribed` (NCCL refuses two ranks on one device: its lines say so).
    N = 1: the same kernels with N local buffers standing in for peers
    (HBM-bound), world sizes 1/2/4/8 emulated. One JSON line per (size, N,
    engine)."""
    import torch.distributed as dist
    from paper_2212_05339_b200 import kernels
    from paper_2212_05339_b200.runtime import shard_length

    world, rank, local, oversub = _dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    peak, src = _peaks()
    sizes = [int(x) for x in args.sweep_sizes.split(",")]
    reps = args.steps
    flush = torch.ones(64 * 2 ** 20, dtype=torch.float32, device=dev)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)
    sc = kernels.new_step_scalars(dev)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=0.0)
    transport = None
    kind = "local"
    if world > 1:
        from paper_2212_05339_b200.transport import IpcTransport, SymmMemTransport, primary_contexts
        kind = "p2p" if args.transport == "p2p" else "ipc"
        transport = SymmMemTransport() if kind == "p2p" else IpcTransport()
    nccl_ok = world > 1 and not oversub and dist.get_backend() == "nccl"

    def timeit(fn, barrier):
        ts = []
        for i in range(reps + 2):
            torch.sum(flush, dim=0, out=flush_sink)
            if barrier is not None:
                barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        return _max_over_ranks(statistics.median(ts), world)

    def emit(rec):
        rec.update({"sweep": "chunk", "world": world, "peers": kind if world > 1 else "local buffers",
                    "hbm_peak_gbs": peak, "reps": reps})
        if oversub:
            rec["oversubscribed"] = oversub
        if rank == 0:
            print(json.dumps(rec), flush=True)

    for mb in sizes:
        C = mb * 2 ** 20 // 2                      # bf16 elements of one chunk
        if world > 1:
            S = shard_length(C, world)
            P = world * S
            g = torch.Generator(device=dev).manual_seed(77 + rank)
            shard = transport.alloc((S,), torch.bfloat16, dev)
            shard.copy_(torch.randn(S, generator=g, device=dev).to(torch.bfloat16))
            block = transport.alloc((P,), torch.bfloat16, dev)
            block.copy_(torch.randn(P, generator=g, device=dev).to(torch.bfloat16))
            g32 = torch.empty(S, device=dev)
            ps = transport.peer_ptrs(shard)
            pb = transport.peer_ptrs(block)
            segs = [p + rank * S * 2 for p in pb]
            bar = transport.device_barrier
            bus = (world - 1) / world * 2 * P      # bytes: the gathered block / the bf16 reduce-scatter input
            for engine, fn in (("k2_fetch_sm", lambda: kernels.fetch(block, ps, S, rank=rank)),
                               ("k2_fetch_ce", lambda: kernels.fetch(block, ps, S, engine="ce", rank=rank)),
                               ("k3_release", lambda: kernels.release(g32, segs, S, torch.bfloat16, 1.0, sc))):
                ms = timeit(fn, bar)
                emit({"chunk_mb": mb, "engine": engine, "shard_elems": S, "ms": ms,
                      "bus_gbs": bus / (ms * 1e-3) / 1e9, "frac_of_900": bus / (ms * 1e-3) / 1e9 / 900})
            if args.sweep_check:
                emit(_sweep_parity_peers(mb, world, rank, S, block, pb, sc, dev, bar))
            if nccl_ok:
                out16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
                blk32 = block.float()
                out32 = torch.empty(S, device=dev)
                for engine, fn, nbytes in (
                        ("nccl_all_gather", lambda: dist.all_gather_into_tensor(block, shard), bus),
                        ("nccl_reduce_scatter_bf16", lambda: dist.reduce_scatter_tensor(out16, block), bus),
                        ("nccl_reduce_scatter_f32", lambda: dist.reduce_scatter_tensor(out32, blk32), 2 * bus)):
                    ms = timeit(fn, bar)
                    emit({"chunk_mb": mb, "engine": engine, "shard_elems": S, "ms": ms,
                          "bus_gbs": nbytes / (ms * 1e-3) / 1e9, "frac_of_900": nbytes / (ms * 1e-3) / 1e9 / 900})
                del out16, blk32, out32
            else:
                for engine in ("nccl_all_gather", "nccl_reduce_scatter_bf16", "nccl_reduce_scatter_f32"):
                    emit({"chunk_mb": mb, "engine": engine, "unavailable":
                          "NCCL needs one GPU per rank" if oversub else "process group is not NCCL"})
            # K4 on this rank's shard (local HBM)
            p32, m, v = (torch.zeros(S, device=dev) for _ in range(3))
            p16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
            g32.normal_()
            tab = kernels.AdamTable([(p32, m, v, g32, p16, S)], dev)
            ms = timeit(lambda: kernels.adam(tab, hp, 1, sc, torch.bfloat16), bar)
            emit({"chunk_mb": mb, "engine": "k4_adam", "shard_elems": S, "ms": ms,
                  "hbm_gbs": 30 * S / (ms * 1e-3) / 1e9, "frac": 30 * S / (ms * 1e-3) / 1e9 / peak})
            del shard, block, g32, p32, m, v, p16, tab
            continue
        # K1: pack a chunk from its members (a GPT-2 layer's 12 parameters in order, cycled, greedy like
        # pack_chunks; 1.3B widths, GPT-2 small's below 24 MB chunks; the unused tail zero-filled) —
        # 2*sum(numel) read + 2*C write
        h = 2048 if C >= 3 * 2048 * 2048 else 768
        layer = [h, h, 3 * h * h, 3 * h, h * h, h, h, h, 4 * h * h, 4 * h, 4 * h * h, h]
        members, off, i = [], 0, 0
        while off + layer[i % 12] <= C and i < 10_000:
            members.append(off)
            off += layer[i % 12]
            i += 1
        if not members:  # the chunk is smaller than a layer's first weight: split the chunk evenly
            members, off = [0], C
            sizes = [C]
        else:
            sizes = [layer[j % 12] for j in range(len(members))]
        pk_src = [torch.randn(n, device=dev).to(torch.bfloat16) for n in sizes]
        pk_dst = torch.empty(C, dtype=torch.bfloat16, device=dev)
        pk = [(t, o) for t, o in zip(pk_src, members)]
        t_k1 = timeit(lambda: kernels.chunk_pack(pk_dst, pk, used_len=off), None)
        k1_bytes = 2 * off + 2 * C
        emit({"chunk_mb": mb, "emulated_world": 1, "engine": "k1_pack", "shard_elems": C, "members": len(pk),
              "ms": t_k1, "hbm_gbs": k1_bytes / (t_k1 * 1e-3) / 1e9, "frac": k1_bytes / (t_k1 * 1e-3) / 1e9 / peak})
        del pk_src, pk_dst, pk
        for w in (1, 2, 4, 8):
            S = shard_length(C, w)
            if args.sweep_graph:
                _sweep_graph_stream(mb, w, S, dev, reps, flush, flush_sink, hp, peak, emit)
                continue
            shards = [torch.randn(S, device=dev).to(torch.bfloat16) for _ in range(w)]
            block = torch.empty(w * S, dtype=torch.bfloat16, device=dev)
            g32 = torch.empty(S, device=dev)
            t_f = timeit(lambda: kernels.fetch(block, [s.data_ptr() for s in shards], S), None)
            t_fc = timeit(lambda: kernels.fetch(block, [s.data_ptr() for s in shards], S, engine="ce"), None)
            # world 1 is the runtime's norm pass (the gradient stays in the chunk: no fp32 output)
            t_r = timeit(lambda: kernels.release(g32 if w > 1 else None, [s.data_ptr() for s in shards], S,
                                                 torch.bfloat16, 1.0, sc), None)
            p32, m, v = (torch.zeros(S, device=dev) for _ in range(3))
            p16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
            if w == 1:
                g32.normal_()   # (at N > 1 K3 wrote it)
            tab = kernels.AdamTable([(p32, m, v, g32, p16, S)], dev)
            t_a = timeit(lambda: kernels.adam(tab, hp, 1, sc, torch.bfloat16), None)
            for engine, ms, nbytes in (("k2_fetch_sm", t_f, 2 * 2 * w * S), ("k2_fetch_ce", t_fc, 2 * 2 * w * S),
                                       ("k3_release", t_r, 2 * w * S + (4 * S if w > 1 else 0)),
                                       ("k4_adam", t_a, 30 * S)):
                emit({"chunk_mb": mb, "emulated_world": w, "engine": engine, "shard_elems": S, "ms": ms,
                      "hbm_gbs": nbytes / (ms * 1e-3) / 1e9, "frac": nbytes / (ms * 1e-3) / 1e9 / peak})
            if args.sweep_check:
                emit(_sweep_parity(mb, w, S, shards, block, dev, hp))
            del shards, block, g32, p32, m, v, p16, tab
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            print(json.dumps({"sweep": "contexts", "rank": rank, "cuda_contexts_on_devices": primary_contexts()}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="gpt2-1.3b")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--sweep-sizes", default="4,8,16,32,64,128,256", help="chunk sizes in MB for --sweep")
    ap.add_argument("--sweep-check", action="store_true",
                    help="--sweep: also check each size's K2/K3 (and at N=1 K4) outputs against the C oracle")
    ap.add_argument("--sweep-graph", action="store_true",
                    help="--sweep at N=1: time each kernel as R back-to-back launches on distinct buffers in one "
                         "CUDA graph (the step's issue pattern) instead of single cold launches")
    ap.add_argument("--plan", default=None, help="plan file under plans/, {n} = world size "
                    "(default <model>_n<N>.json), e.g. gpt2-4b_offload_n{n}.json")
    ap.add_argument("--batch", type=int, default=0,
                    help="per-rank micro-batch (default: the preset's 8, BASELINE.json's configuration); a smaller "
                         "one only for functional runs of many ranks on one GPU")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing parity check against the oracle")
    ap.add_argument("--cpu-update", choices=["split", "host", "stream"], default="split",
                    help="CPU-home chunk update: host threads, GPU-streamed, or split by measured rate")
    ap.add_argument("--recompute", choices=["auto", "on", "off"], default="auto",
                    help="activation checkpointing: on = recompute each node in the backward (the reference's "
                         "design), off = keep the forward graphs, auto = off when every chunk stays resident "
                         "and the activations fit in HBM")
    ap.add_argument("--deterministic", action="store_true",
                    help="deterministic library algorithms (cuDNN attention's deterministic backward): the whole "
                         "step becomes run-to-run bit-reproducible (our kernels always are)")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=True,
                    help="every chunk GPU-home, world 1 or --transport ipc: capture the whole step as one CUDA graph")
    ap.add_argument("--overlap", action="store_true",
                    help="issue the GPU update per chunk on an optimizer stream under the next forward")
    ap.add_argument("--transport", choices=["auto", "nccl", "p2p", "ipc", "ipc-ce"],
                    default=os.environ.get("ELX_TRANSPORT", "auto"),
                    help="N>1 fetch/release path: auto (default) = in-kernel P2P over our CUDA-IPC mappings when every "
                         "peer GPU is reachable, else NCCL; nccl = NCCL collectives + K3; ipc / ipc-ce = K2 on SMs / "
                         "copy engines over IPC mappings; p2p = over torch symmetric memory")
    args = ap.parse_args()
    if args.deterministic:
        os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
        torch.backends.cudnn.deterministic = True
        torch.use_deterministic_algorithms(True)
    if args.warmup < 3 and not args.sweep and args.impl == "ours":
        print("warning: --warmup < 3 is below the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sweep(args) if args.sweep else run_ours(args)
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            # no rank exits (releasing the CUDA-IPC memory it exported) while a peer still maps it
            torch.cuda.synchronize()
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
