# div6 (fp32 3-D division): exhaustive check, 3-D parity, stencil7 A/B vs HEAD (.ab_old)
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rA -k "div20 or stencil7 or edge or 3d" 2>&1 | grep -E "PASS|FAIL|passed|failed|Error" > gpurun_out/o/pytest.log
for i in 1 2 3; do
  (cd .ab_old && HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil7 --steps 30 --no-cpu-baseline --no-e2e) > gpurun_out/o/s7_old.$i.json 2>/dev/null
  HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil7 --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/o/s7_new.$i.json 2>/dev/null
done
cat gpurun_out/o/pytest.log
for f in gpurun_out/o/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
