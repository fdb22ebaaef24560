# LU panel diagnostics: per-phase panel traces (both kernels) and whole-factorization timings
tr() { python tools/panel_trace.py 16384 0 8192 14336 16256 2>&1 | grep -E "panel trace|Error|error" | sed -E 's/\[poller kernel[^]]*\]//' | head -4; }
echo "== default"; tr
echo "== cta-synchronous kernel only"; DENSOLVE_PANEL_KERNEL=2 tr
for cfg in "DENSOLVE_PANEL_KERNEL=2" "DENSOLVE_PANEL_KERNEL=0"; do
  echo "== $cfg"; env $cfg python tools/lu_var.py 16384 3 2>&1 | tail -1; env $cfg python tools/lu_var.py 32768 2 2>&1 | tail -1
done
