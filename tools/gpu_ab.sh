DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_tkT2.so timeout 300 python tools/probes/tk_trace2.py > gpurun_out/tk_trace2.log 2>&1; echo "rc=$?"; cat gpurun_out/tk_trace2.log | tail -20
