#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines (HV720 default, reference arm,
# Wan720, sparsity sweep), ncu launch list, the K1/K5 seams and one ncu --set
# full capture of K4. Outputs under gpurun_out/. STAGES selects a subset.
set -u
mkdir -p gpurun_out
STAGES=${STAGES:-"test smoke bench ref sweep seams launches full"}
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for s in $STAGES; do
  case $s in
    test) timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log ;;
    headpar) timeout 600 python -m pytest tests/test_gpu_headpar.py -q -p no:cacheprovider > gpurun_out/pytest_headpar.log 2>&1; echo "headpar rc=$?"; tail -2 gpurun_out/pytest_headpar.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log ;;
    ref) timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log ;;
    sweep)
      for sp in 0.5 0.75 0.95; do timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --sparsity $sp > gpurun_out/bench_hv720_$sp.log 2>&1; echo "sweep $sp rc=$?"; done
      timeout 900 python bench.py --config wan720 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_wan720.log 2>&1; echo "wan720 rc=$?"
      timeout 900 python bench.py --config hv720_8x16 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_hv720_8x16.log 2>&1; echo "8x16 rc=$?"
      timeout 900 python bench.py --data smooth --steps 5 --warmup 3 --no-cpu --no-dense > gpurun_out/bench_hv720_smooth.log 2>&1; echo "smooth rc=$?" ;;
    seams) timeout 300 python tools/probes/seam_k1k5.py > gpurun_out/seams.log 2>&1; echo "seams rc=$?"; cat gpurun_out/seams.log | tail -1
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:permute -c 4 --csv --log-file gpurun_out/seams_ncu.csv python tools/probes/seam_k1k5.py --reps 1 > /dev/null 2>&1; echo "seams ncu rc=$?" ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 2 -c 1 -f -o gpurun_out/k4 python bench.py --steps 1 --warmup 3 --no-cpu --no-dense > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?" ;;
  esac
done
