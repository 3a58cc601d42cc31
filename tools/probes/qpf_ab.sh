# lane-half K4: prefetch of the next item's Q rows into L2 (LH_Q_PREFETCH) on / off, interleaved
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
for r in 1 2; do
  for fl in "-DLH_Q_PREFETCH=0" ""; do
    DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run "[$fl]"
  done
done
