# lane-half K4 build variants, interleaved: default / sleeping waits / no polynomial exps / half polynomial
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
for r in 1 2; do
  for fl in "" "-DDA_LH_SLEEP" "-DLH_POLY_EVERY=0" "-DLH_POLY_EVERY=2"; do
    DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run "[$fl]"
  done
done
