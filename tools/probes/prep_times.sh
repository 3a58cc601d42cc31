# per-kernel device times of one HV720 pipeline call (ncu launch list)
python -m paper_2505_14708_b200.build >/dev/null 2>&1
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/prep.csv python tools/probes/k4_ab.py --data gaussian --reps 1 >/dev/null 2>&1
echo "ncu rc=$?"
