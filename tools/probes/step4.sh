python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 300 python tools/probes/dbg_k4.py 2>&1 | grep -E "max err|rerun|count"
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "seam or tcgen05 or extreme or zero_sparsity or 720p or host" 2>&1 | tail -2
timeout 300 python tools/probes/k4_ab.py
DA_NVCC_FLAGS="-DDA_TRACE" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
timeout 300 python tools/probes/k4_trace3.py | tail -8
