#!/bin/bash
# compute-sanitizer passes over the cooperative / persistent / TMA kernels:
# racecheck + synccheck on smoke() (persistent stage 1, persistent IPM, surface kernels)
# and on small TMA product shapes; memcheck on the same.  Logs under gpurun_out/.
out=gpurun_out
mkdir -p $out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  timeout 900 $S --tool $tool --error-exitcode 9 --kernel-name-exclude regex:at:: \
    python -c "import __graft_entry__ as g; g.smoke()" > $out/sanitize_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?"
  timeout 900 $S --tool $tool --error-exitcode 9 \
    python -m pytest -q -x tests/test_gpu_tma.py -k "4100-2050-10 or 4100-2050-5 or 4097" \
    > $out/sanitize_tma_$tool.log 2>&1
  echo "tma $tool rc=$?"
done
