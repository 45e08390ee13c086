# 3-D kernel: 3-way rotated z loop, hoisted predicates, one division range check per float4 — A/B vs HEAD
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/am
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py -q -p no:cacheprovider -rA -k "div20 or stencil7 or 3d or edge" 2>&1 | grep -E "PASS|FAIL|passed|failed|Error|mismatch" > gpurun_out/am/pytest.log
for i in 1 2; do for st in 30 100; do
  (cd .ab_old && HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil7 --steps $st --no-cpu-baseline --no-e2e) > gpurun_out/am/s7_old_$st.$i.json 2>/dev/null
  HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil7 --steps $st --no-cpu-baseline --no-e2e > gpurun_out/am/s7_new_$st.$i.json 2>/dev/null
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed.avg.pct_of_peak_sustained_active --clock-control none -k regex:stencil7_kernel -s 5 -c 1 --csv python bench.py --workload stencil7 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/am/ncu_new.csv 2>/dev/null
cat gpurun_out/am/pytest.log
for f in gpurun_out/am/*.json; do printf "%-22s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
grep -h "inst_executed\|duration" gpurun_out/am/ncu_new.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
