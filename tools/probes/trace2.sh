for fl in "-DDA_CRIT_SLEEP" ""; do
DA_NVCC_FLAGS="-DDA_TRACE $fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
echo "flags: $fl"
timeout 300 python tools/probes/k4_trace.py 24 | tail -13
DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 300 python tools/probes/k4_ab.py --data gaussian
done
