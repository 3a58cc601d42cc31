#!/bin/bash
# Quick GPU check after a change: shard tests, sanitizers over every device
# path (tools/sanitize.py), the default bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_shards.log 2>&1; echo "shards rc=$?"; tail -1 gpurun_out/pytest_shards.log
bash tools/gpu_sanitize.sh
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
