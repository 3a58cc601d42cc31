# lane-half K4: per-half Q ownership (current file) vs the previous version (tools/probes/tmp/attn_lh_old.cu)
cp paper_2505_14708_b200/csrc/attn_lh.cu /tmp/attn_lh_cur.cu
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run new
  cp tools/probes/tmp/attn_lh_old.cu paper_2505_14708_b200/csrc/attn_lh.cu
  python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run old
  cp /tmp/attn_lh_cur.cu paper_2505_14708_b200/csrc/attn_lh.cu
done
DA_NVCC_FLAGS="-DLH_PROF" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; python tools/probes/lh_prof.py
