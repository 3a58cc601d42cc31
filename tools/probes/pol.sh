python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for pol in 0 1 2 4 6 7; do echo "DA_L2POL=$pol"; DA_L2POL=$pol timeout 300 python tools/probes/k4_ab.py --data gaussian; done
