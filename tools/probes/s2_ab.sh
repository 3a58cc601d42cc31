# lane-half K4: two S buffers per half (O single) vs one (O double), interleaved; GPU suite on the default
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  for fl in "-DLH_S2=0" ""; do
    DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run "[$fl]"
  done
done
DA_NVCC_FLAGS="-DLH_PROF" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; python tools/probes/lh_prof.py
