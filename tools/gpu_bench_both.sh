#!/bin/bash
# Both bench arms the way the driver runs them (reference first), plus the GPU tests.
# Usage (under gpurun): bash tools/gpu_bench_both.sh TAG [K W]
tag=${1:-r02}; K=${2:-20}; W=${3:-5}
out=gpurun_out; mkdir -p $out
( time timeout 1700 python bench.py --impl reference --gpus 1 --steps $K --warmup $W ) > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
echo "ref exit $?"; tail -c 1500 $out/bench_ref_$tag.json; tail -4 $out/bench_ref_$tag.err
( time timeout 1700 python bench.py --gpus 1 --steps $K --warmup $W ) > $out/bench_$tag.json 2> $out/bench_$tag.err
echo "bench exit $?"; tail -c 6000 $out/bench_$tag.json; tail -4 $out/bench_$tag.err
