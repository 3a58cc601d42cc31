DA_NVCC_FLAGS="-DDA_TRACE" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
for fk in 4 7; do echo "DA_FAKELOAD=$fk"; DA_FAKELOAD=$fk timeout 300 python tools/probes/k4_ab.py --data gaussian; DA_FAKELOAD=$fk timeout 300 python tools/probes/k4_trace.py 24 | tail -5; done
