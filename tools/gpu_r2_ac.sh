# GEMM before (0812bc8, .ab_old) vs after the KGate/segment restructuring: bench + DRAM bytes
O=gpurun_out/ac; mkdir -p $O
for i in 1 2; do
  (cd .ab_old && HDA_AUTOBUILD=0 timeout 300 python bench.py --workload gemm --no-cpu-baseline --no-e2e) > $O/gemm_old.$i.json 2>/dev/null
  HDA_AUTOBUILD=0 timeout 300 python bench.py --workload gemm --no-cpu-baseline --no-e2e > $O/gemm_new.$i.json 2>/dev/null
done
for v in old new; do
  d=.; [ $v = old ] && d=.ab_old
  (cd $d && HDA_AUTOBUILD=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm2_kernel -s 4 -c 3 --csv python bench.py --workload gemm --steps 3 --warmup 3 --no-cpu-baseline --no-e2e) > $O/ncu_$v.csv 2>/dev/null
done
for f in $O/*.json; do printf "%-20s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
grep -h "gemm2" $O/ncu_*.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -20
