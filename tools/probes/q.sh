python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/probes/dbg_k4.py
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "seam or tcgen05 or extreme or zero_sparsity or 720p" 2>&1 | tail -8
