mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in pair transposed; do DA_K4=$v timeout 300 python tools/probes/k4_ab.py >> gpurun_out/ab.log 2>&1; done
cat gpurun_out/ab.log
