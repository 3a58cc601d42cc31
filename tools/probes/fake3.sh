# K4 with parts of its work skipped (DA_FAKELOAD bits: 1 K copies, 2 V copies, 4 softmax)
python -m paper_2505_14708_b200.build >/dev/null 2>&1
for fk in ${FKS:-0 1 2 3 4 7}; do echo "DA_FAKELOAD=$fk"; DA_FAKELOAD=$fk timeout 300 python tools/probes/k4_ab.py --data gaussian --reps 5 2>&1 | tail -2; done
