# lane-half K4: L2 cache-policy hints (LH_L2POL bits), interleaved
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
for r in 1 2; do
  for fl in "" "-DLH_L2POL=6" "-DLH_L2POL=7"; do
    DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run "[$fl]"
  done
done
