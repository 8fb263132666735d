#!/bin/bash
# Launch list of the bench's timed region and ncu --set full captures of the c4 products.
# Run on the GPU box (gpurun) after `python bench.py` has exited 0 without ncu.
#   bash scripts/profile_c4.sh <tag>
set -u
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
# 1. kernels launched inside bench.py's timed region only (NVTX range "bench_timed")
ncu --nvtx --nvtx-include "bench_timed/" --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $out/${tag}_c4_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-aux --no-cpu > $out/${tag}_c4_launches.log 2>&1
echo "launch list rc=$?"
# 2. full sections of the streaming products (cold cache, serialised)
ncu --set full --clock-control none --import-source on \
    -k regex:"k_rowprod|k_colprod|k_dualprod" -c 6 -f -o $out/${tag}_ncu_products_c4 \
    python scripts/c4_sweeps.py 3 4 > $out/${tag}_ncu_products_c4.log 2>&1
echo "ncu products rc=$?"
