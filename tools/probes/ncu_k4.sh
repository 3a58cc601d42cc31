# one ncu --set full capture of the K4 kernel on the HV720 bench workload
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 2 -c 1 -f -o gpurun_out/${NCU_NAME:-k4} python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
