# lane-half K4: V by cp.async (LSU) next to K bulk copies vs both bulk; interleaved; then the GPU suite on cp.async
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
for r in 1 2; do
  for fl in "" "-DLH_V_CPASYNC=1"; do
    DA_NVCC_FLAGS="$fl" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run "[$fl]"
  done
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
