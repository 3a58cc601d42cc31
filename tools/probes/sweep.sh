# bench lines for the other configs (Wan720 at 75 %, the HV720 sparsity sweep), with dense SDPA
for a in "--config wan720" "--sparsity 0.5" "--sparsity 0.75" "--sparsity 0.95"; do
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu --dense 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$a', d['config']['workload'], 'ms', round(d['value'], 2), 'dense', round(d.get('dense_sdpa_ms', 0), 1), 'x', round(d.get('speedup_vs_dense_sdpa', 0), 2), 'frac', round(d['roofline']['frac'], 3), 'e2e', round(d['e2e']['value'], 1))"
done
