timeout 600 python tools/probes/k4_variants.py run tk lh --rounds 2 > gpurun_out/k4_tk.log 2>&1
tail -4 gpurun_out/k4_tk.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_tk.log 2>&1
tail -15 gpurun_out/pytest_tk.log
