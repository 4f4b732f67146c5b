"""CPU oracle for the Elixir chunk-memory hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (and ``bench.py --impl reference``) may import, link or execute anything
in this package, and only as the checker or the timed CPU reference — never
as part of the product path (``paper_2212_05339_b200`` never imports it).

Contents
  layout_ref.py  pure-Python restatement of the reference's layout and
                 schedule functions (offplan/chunking.py, rcache_sim.py,
                 profiles.py), cited line by line. PINNED: checked against the
                 golden vectors generated from the reference itself
                 (tests/golden/make_golden.py) and against the reference's own
                 known-answer tests (tests/test_oracle_layout.py).
  arith.py       numpy restatement of the floating-point / byte side of the
                 path: chunk pack, fetch (all-gather), release (rank-ordered
                 fp32 reduce x inv_scale, sum of squares, overflow), AdamW,
                 clip coefficient. The reference contains NO implementation
                 of any of these: the arithmetic is "parity
                 unpinned" by the reference. It is pinned instead against
                 torch.optim.AdamW (single-tensor path, torch 2.11 CPU) and
                 torch.nn.utils.clip_grad_norm_ via committed fixtures
                 (tests/golden/adamw_golden.npz).
  c/elx_oracle.c plain-C restatement of arith.py (OpenMP), used as the timed
                 CPU baseline at full size; cross-checked against arith.py.
  gpt2_ref.py    the GPT-2 layer in stock torch ops (the CPU baseline's model
                 math; the product's layer runs our CUDA kernels).
"""
