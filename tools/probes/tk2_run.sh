DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkP.so timeout 300 python tools/probes/tk_prof.py > gpurun_out/tk2_prof.log 2>&1; echo "prof rc=$?"; tail -26 gpurun_out/tk2_prof.log
DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkT.so timeout 300 python tools/probes/tk_trace.py > gpurun_out/tk2_trace.log 2>&1; echo "trace rc=$?"; cat gpurun_out/tk2_trace.log | tail -30
