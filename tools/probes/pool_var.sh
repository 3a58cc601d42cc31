# pool_avg_kernel variants: rows per batch x min blocks per SM
for cfg in "4 4" "8 3" "2 4" "8 4" "4 3"; do set -- $cfg
  DA_NVCC_FLAGS="-DDA_POOL_RB=$1 -DDA_POOL_MINB=$2" python -m paper_2505_14708_b200.build --force >/dev/null 2>&1
  echo -n "RB=$1 MINB=$2 "; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pool_avg -c 1 python tools/probes/k4_ab.py --data gaussian --reps 1 2>&1 | grep gpu__time
done
