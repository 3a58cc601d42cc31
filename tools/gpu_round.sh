#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list and one
# ncu --set full capture of K4. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
STAGES=${STAGES:-"test smoke bench launches full"}
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for s in $STAGES; do
  case $s in
    test) timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 900 python bench.py --steps 10 --warmup 3 --dense > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 2 -c 1 -f -o gpurun_out/k4 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?" ;;
  esac
done
