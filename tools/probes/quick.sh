# quick GPU check: gpu tests + K4 A/B on gaussian/smooth
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 300 python tools/probes/k4_ab.py ${AB_ARGS:-}
