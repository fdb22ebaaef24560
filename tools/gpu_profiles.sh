#!/bin/bash
# Refresh the ncu evidence under gpurun_out/ (then summarised into profiles/):
#   launch lists (gpu__time_duration.sum, --clock-control none) of the bench headline command,
#   of LU n=16384, Cholesky n=16384 and of one GMRES(30) C2 cycle; --set full captures of the GEMV
#   (bench n), the K=512 trailing GEMM, one LU panel launch of each kernel and the GMRES cluster step.
tag=${1:-s3}
out=gpurun_out
mkdir -p $out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $out/launches_bench_$tag.csv python bench.py --steps 1 --warmup 3 --only-cg --no-cpu-baseline \
  > $out/ncu_bench_$tag.log 2>&1; echo "bench list $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_lu_$tag.csv python tools/profile_run.py lu 16384 > /dev/null 2>&1; echo "lu list $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_gmres_$tag.csv python tools/profile_run.py gmres 4096 > /dev/null 2>&1; echo "gmres list $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_chol_$tag.csv python tools/profile_run.py chol 16384 > /dev/null 2>&1; echo "chol list $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:arnoldi_orth_cluster -s 25 -c 1 \
  -o $out/orth_full_$tag -f python tools/profile_run.py gmres 4096 > /dev/null 2>&1; echo "orth full $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lu_panel_warp -s 10 -c 1 \
  -o $out/panelw_full_$tag -f python tools/profile_run.py lu 16384 > /dev/null 2>&1; echo "poller panel full $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:colstream_mv -s 2 -c 1 \
  -o $out/gemv_full_$tag -f python tools/profile_run.py gemv 32768 > /dev/null 2>&1; echo "gemv full $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm64 -s 1 -c 1 \
  -o $out/gemm_full_$tag -f python tools/profile_run.py gemm 16384 16384 512 > /dev/null 2>&1; echo "gemm full $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lu_panel -s 40 -c 1 \
  -o $out/panel_full_$tag -f python tools/profile_run.py lu 16384 > /dev/null 2>&1; echo "panel full $?"
for f in $out/launches_*_$tag.csv; do python tools/launch_summary.py $f | head -12; done
