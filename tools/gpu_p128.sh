#!/bin/bash
# 8x16 pools (p = 128) on tcgen05: full GPU suite, the hv720_8x16 bench line, the default line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config hv720_8x16 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_8x16.log 2>&1; echo "8x16 rc=$?"; tail -1 gpurun_out/bench_8x16.log | cut -c1-300
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-dense > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-200
