# K4 lane-half variant (DA_K4=lh): correctness smoke, GPU suite, A/B timing against the pair kernel
python -m paper_2505_14708_b200.build >/dev/null 2>&1
DA_K4=lh timeout 120 python tools/probes/k4small.py 2>&1 | tail -1
DA_K4=lh timeout 120 python tools/probes/k4hv.py 2>&1 | tail -1
timeout 120 python tools/probes/k4hv.py 2>&1 | tail -1
DA_K4=lh timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for r in 1 2; do for v in pair lh; do echo -n "$v "; DA_K4=$v timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 7 2>&1 | tail -1; done; done
