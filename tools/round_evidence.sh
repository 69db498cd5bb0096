#!/bin/bash
# End-of-round evidence on one B200: bench line (plain, then torchrun N=1), reference arm, per-config
# table, then the ncu passes of tools/ncu_capture.sh (each only after its command exited 0 without ncu).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-c128 > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err
echo "torchrun rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python tools/bench_configs.py --json gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
bash tools/ncu_capture.sh > gpurun_out/ncu_capture.log 2>&1; echo "ncu rc=$?"
