timeout 600 python tools/probes/k4_variants.py run lhold lhnew3 --rounds 3 > gpurun_out/k4_lh_ring3.log 2>&1; echo "ab rc=$?"; tail -2 gpurun_out/k4_lh_ring3.log
bash tools/gpu_sanitize.sh
STAGES="test" bash tools/gpu_round.sh
