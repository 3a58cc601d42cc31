# lane-half K4: K / V ring depth split (LH_KSL / LH_VSL slots of two tiles), interleaved
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
for r in 1 2; do
  for fl in "" "-DLH_KSL=4 -DLH_VSL=2" "-DLH_KSL=2 -DLH_VSL=4"; do
    DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run "[$fl]"
  done
done
