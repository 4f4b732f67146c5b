#!/usr/bin/env bash
# The N > 1 measurements this environment cannot make (one GPU per call), as one command for a node with
# 2-8 B200s. Writes everything under gpurun_out/multigpu/; summarise into profiles/ after.
#
#   bash scripts/multigpu_campaign.sh [max_gpus]
#
# 1. the configs[4] chunk sweep on real peer pointers (K2 SM/CE, K3) beside NCCL all-gather / reduce-scatter,
#    with the register-staged A/B of the peer reads (ELX_K3_PEER_TMA=0 ELX_K2_TMA=-1);
# 2. the hardware profile's n-GPU rows (b_g2g from K2 on NVLink peers, per-n b_c2g / b_g2c / v_g / v_c);
# 3. the GPT-2 1.3B step at N = 2/4/8 per transport (ipc default, ipc-ce, p2p, nccl), each line with the
#    whole-step parity check on every rank;
# 4. the distinct-GPU tests (tests/test_multigpu.py).
set -u
MAX=${1:-$(python -c "import torch; print(torch.cuda.device_count())")}
OUT=gpurun_out/multigpu
mkdir -p "$OUT"
run() {  # run <n> <tag> <args...>
  local n=$1 tag=$2; shift 2
  timeout 3600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) "$@" > "$OUT/$tag.jsonl" 2> "$OUT/$tag.err"
}
for n in 2 4 8; do
  [ "$n" -le "$MAX" ] || continue
  run "$n" "sweep_n$n" bench.py --sweep --gpus "$n" --steps 20
  ELX_K3_PEER_TMA=0 ELX_K2_TMA=-1 run "$n" "sweep_regstaged_n$n" bench.py --sweep --gpus "$n" --steps 20
  run "$n" "profile_hw_n$n" scripts/profile_hw.py
  for tr in ipc ipc-ce p2p nccl; do
    run "$n" "bench_${tr}_n$n" bench.py --gpus "$n" --transport "$tr" --steps 10 --warmup 3 --no-cpu
  done
done
timeout 3600 python -m pytest tests/test_multigpu.py -q > "$OUT/test_multigpu.txt" 2>&1
echo "done: $OUT"
