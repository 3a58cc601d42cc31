DA_NVCC_FLAGS="-DDA_TRACE -DTRACE_T=160" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 300 python tools/probes/k4_trace2.py 5
DA_NVCC_FLAGS="-DDA_TRACE -DTRACE_T=128" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 300 python tools/probes/k4_trace2.py 4 | tail -8
