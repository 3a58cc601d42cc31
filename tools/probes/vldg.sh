python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for vl in 0 1; do echo "DA_VLDG=$vl"; DA_VLDG=$vl timeout 300 python tools/probes/dbg_k4.py 2>&1 | grep -E "max err|rerun"; DA_VLDG=$vl timeout 300 python tools/probes/k4_ab.py; done
DA_VLDG=1 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "seam or tcgen05 or extreme or zero_sparsity or 720p" 2>&1 | tail -3
