#!/bin/bash
# One GPU session: GPU tests, the bench line, and the ncu launch list of the same bench command.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu_$tag.log
tail -3 $out/pytest_gpu_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?"
tail -c 3000 $out/bench_$tag.json
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > $out/bench_ref_$tag.json 2>&1; echo "ref exit $?"
tail -c 1500 $out/bench_ref_$tag.json
