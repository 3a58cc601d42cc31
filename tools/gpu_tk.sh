#!/bin/bash
# The transposed TMEM-fed K4 experiment (profiles/r02/tk/README.md) on one box:
# build the variants here first (no GPU needed):
#   python tools/probes/k4_variants.py build lh tk=-DDA_K4_TK tkP=-DDA_K4_TK,-DTK_PROF tkT=-DDA_K4_TK,-DTK_TRACE
# then run this script through gpurun. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 600 python tools/probes/k4_variants.py run lh tk --rounds 2 > gpurun_out/k4_tk_ab.log 2>&1; echo "ab rc=$?"; tail -2 gpurun_out/k4_tk_ab.log
DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkP.so timeout 300 python tools/probes/tk_prof.py > gpurun_out/tk_prof.log 2>&1; echo "prof rc=$?"
DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkT.so timeout 300 python tools/probes/tk_trace.py > gpurun_out/tk_trace.log 2>&1; echo "trace rc=$?"
# parity of the experimental kernel: the whole GPU suite through the tk library
DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tk.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_tk.log 2>&1; echo "pytest tk rc=$?"; tail -2 gpurun_out/pytest_tk.log
