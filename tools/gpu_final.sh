# Round-end evidence: GPU tests, the bench line (+ force-sharded), launch lists of the
# headline, LU and GMRES C2, and full captures of the GEMV, the K=512 TMA GEMM and the
# persistent (SM-reserving) LU trailing GEMM.
tag=${1:-r02f}
out=gpurun_out; mkdir -p $out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest_gpu_$tag.log
t0=$(date +%s); timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench exit $? ($(( $(date +%s) - t0 )) s)"
timeout 300 python bench.py --force-sharded --only-cg --steps 5 --warmup 3 > $out/bench_fs_$tag.json 2>/dev/null; echo "fs exit $?"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $out/launches_bench_$tag.csv \
  python bench.py --steps 1 --warmup 3 --only-cg --no-cpu-baseline > /dev/null 2>&1; echo "list bench $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_lu_$tag.csv \
  python tools/profile_run.py lu 16384 > /dev/null 2>&1; echo "list lu $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_gmres_$tag.csv \
  python tools/profile_run.py gmres 4096 > /dev/null 2>&1; echo "list gmres $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:colstream_mv -s 2 -c 1 \
  -o $out/gemv_full_$tag -f python tools/profile_run.py gemv 32768 > /dev/null 2>&1; echo "gemv full $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm64 -s 1 -c 1 \
  -o $out/gemm_full_$tag -f python tools/profile_run.py gemm 16384 16384 512 > /dev/null 2>&1; echo "gemm full $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm64_tma_persist -s 3 -c 1 \
  -o $out/gemm_persist_full_$tag -f python tools/profile_run.py lu 16384 > /dev/null 2>&1; echo "persist gemm full $?"
for f in $out/launches_*_$tag.csv; do python tools/launch_summary.py $f | head -14; done
