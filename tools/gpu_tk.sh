#!/bin/bash
# K4 A/B (lane-half vs transposed TMEM-fed) and one ncu --set full capture of
# the tk kernel with source-level sampling. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
STAGES=${STAGES:-"ab ncu"}
for s in $STAGES; do
  case $s in
    ab) timeout 600 python tools/probes/k4_variants.py run lh tk --rounds 2 > gpurun_out/k4_ab.log 2>&1; echo "ab rc=$?"; tail -2 gpurun_out/k4_ab.log ;;
    ncu) DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tk.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_tk -s 1 -c 1 -f -o gpurun_out/k4tk python bench.py --steps 1 --warmup 3 --no-cpu --no-dense > gpurun_out/ncu_tk.log 2>&1; echo "ncu tk rc=$?" ;;
    ncu_lh) DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_lh.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_lh -s 1 -c 1 -f -o gpurun_out/k4lh python bench.py --steps 1 --warmup 3 --no-cpu --no-dense > gpurun_out/ncu_lh.log 2>&1; echo "ncu lh rc=$?" ;;
  esac
done
