# K4: dynamic (atomic counter) vs static item scheduling, interleaved A/B/A/B
python -m paper_2505_14708_b200.build >/dev/null 2>&1
for r in 1 2 3; do for s in 0 1; do echo -n "DA_STATIC=$s "; DA_STATIC=$s timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; done; done
