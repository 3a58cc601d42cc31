# K4 under L2 cache-policy variants (DA_L2POL bits: 1 K/V tiles evict_last, 2 Q evict_first, 4 O evict_first)
python -m paper_2505_14708_b200.build >/dev/null 2>&1
for pol in ${POLS:-0 1 2 4 6 7 0}; do echo "DA_L2POL=$pol"; DA_L2POL=$pol timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 5 2>&1 | tail -1; done
