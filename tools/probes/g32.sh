for fl in ""; do
DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:draft32 -c 1 python tools/probes/k4_ab.py --data gaussian --reps 1 2>&1 | grep -E "gpu__time" | sed "s/^/$fl /"
done
