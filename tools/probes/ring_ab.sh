# K4 A/B: current (dynamic, item ring) vs the pre-ring static kernel (tools/probes/tmp/attn_pair_old.cu)
cp paper_2505_14708_b200/csrc/attn_pair.cu /tmp/attn_pair_cur.cu
run() { echo -n "$1 "; timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; }
for r in 1 2; do
  python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run dyn
  cp tools/probes/tmp/attn_pair_old.cu paper_2505_14708_b200/csrc/attn_pair.cu
  python -m paper_2505_14708_b200.build --force >/dev/null 2>&1; run old_static
  cp /tmp/attn_pair_cur.cu paper_2505_14708_b200/csrc/attn_pair.cu
done
