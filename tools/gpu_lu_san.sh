timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash tools/gpu_sanitize.sh
python tools/lu_var.py 16384 3 2>&1 | tail -1
python tools/gmres_rate.py 4096 30 2>&1 | grep cluster | tail -1
