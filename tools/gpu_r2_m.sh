# div20 (constant-reciprocal Markstein fp64 division): exactness, parity, 9-point A/B vs HEAD (.ab_old)
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/m
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "div20 or stencil or config or edge or tma or eigen" > gpurun_out/m/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/m/pytest.log
for i in 1 2 3; do
  (cd .ab_old && HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e) > gpurun_out/m/s9_old.$i.json 2>/dev/null
  HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/m/s9_new.$i.json 2>/dev/null
done
for t in 0; do
  (cd .ab_old && HDA_TMA=$t HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e) > gpurun_out/m/s9_old_tma$t.json 2>/dev/null
  HDA_TMA=$t HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/m/s9_new_tma$t.json 2>/dev/null
done
tail -n 3 gpurun_out/m/pytest.log
for f in gpurun_out/m/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
