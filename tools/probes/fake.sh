python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for fk in 1 3; do echo "DA_FAKELOAD=$fk"; DA_FAKELOAD=$fk timeout 300 python tools/probes/k4_ab.py --data gaussian; done
