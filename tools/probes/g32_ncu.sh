python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:draft32 -c 1 -o gpurun_out/g32 python tools/probes/k4_ab.py --data gaussian --reps 1 > /dev/null 2>&1
ls -la gpurun_out/g32*
