timeout 600 python tools/probes/k4_variants.py run lhnew3 tkI --rounds 2 > gpurun_out/k4_ab8.log 2>&1; echo "ab rc=$?"; grep -v "^ " gpurun_out/k4_ab8.log | tail -3
DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkIP.so timeout 300 python tools/probes/tk_prof.py > gpurun_out/tk_prof_I.log 2>&1; echo "prof rc=$?"; tail -26 gpurun_out/tk_prof_I.log
DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkIT.so timeout 300 python tools/probes/tk_trace.py > gpurun_out/tk_trace_I.log 2>&1; echo "trace rc=$?"; head -14 gpurun_out/tk_trace_I.log
