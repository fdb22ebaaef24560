#!/bin/bash
# One GPU session: GPU tests, the bench line, the reference arm, and the ncu evidence
# (launch list of the bench command + one --set full capture of the dominant kernel).
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag] [phases]
#   phases: any of t (tests) b (bench) r (reference arm) l (launch lists) f (ncu full); default "tbrlf"
tag=${1:-r01}
ph=${2:-tbrlf}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi_$tag.txt 2>&1
if [[ $ph == *t* ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu_$tag.log
  tail -3 $out/pytest_gpu_$tag.log
fi
if [[ $ph == *b* ]]; then
  timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $?"
  tail -c 3000 $out/bench_$tag.json
fi
if [[ $ph == *r* ]]; then
  timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > $out/bench_ref_$tag.json 2>&1; echo "ref exit $?"
  tail -c 1500 $out/bench_ref_$tag.json
fi
NCU=/usr/local/cuda/bin/ncu
if [[ $ph == *l* ]]; then
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file $out/launches_bench_$tag.csv \
    python bench.py --steps 1 --warmup 3 --only-cg --no-cpu-baseline > $out/ncu_bench_$tag.log 2>&1
  echo "ncu launch list exit $?"
  python tools/launch_summary.py $out/launches_bench_$tag.csv | head -20
  timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches_lu_$tag.csv python tools/profile_run.py lu 16384 > $out/ncu_lu_$tag.log 2>&1
  echo "ncu lu exit $?"
  python tools/launch_summary.py $out/launches_lu_$tag.csv | head -20
fi
if [[ $ph == *f* ]]; then
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:colstream_mv -s 2 -c 1 \
    -o $out/gemv_full_$tag -f python tools/profile_run.py gemv 32768 > $out/ncu_full_$tag.log 2>&1
  echo "ncu full gemv exit $?"
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gemm64 -s 10 -c 1 \
    -o $out/gemm_full_$tag -f python tools/profile_run.py lu 16384 > $out/ncu_fullgemm_$tag.log 2>&1
  echo "ncu full gemm exit $?"
fi
