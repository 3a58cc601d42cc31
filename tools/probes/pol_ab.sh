# K4 L2 eviction-policy variants: event-timed A/B, then DRAM bytes per K4 launch (ncu)
timeout 900 python tools/probes/k4_variants.py run pol0 pol3 pol6 pol7 --rounds 2 > gpurun_out/k4_pol.log 2>&1; echo "ab rc=$?"; tail -4 gpurun_out/k4_pol.log
for v in pol0 pol3 pol6 pol7; do
  DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:sparse_attn_lh -c 1 --csv --log-file gpurun_out/pol_$v.csv python tools/probes/sel_once.py > /dev/null 2>&1
  echo "== $v"; grep -o '"\(gpu__time_duration.sum\|dram__bytes_read.sum\|dram__bytes_write.sum\|lts__t_sector_hit_rate.pct\)","[^"]*","[^"]*"' gpurun_out/pol_$v.csv
done
