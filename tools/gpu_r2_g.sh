# A/B: HEAD's TMA consumer (.ab_old, built from the last commit) vs the restructured one
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/g
for i in 1 2 3; do
  (cd .ab_old && HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e) > gpurun_out/g/s9_old.$i.json 2>/dev/null
  HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/g/s9_new.$i.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "edge_values or tma" > gpurun_out/g/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g/pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d_tma -s 6 -c 1 -o gpurun_out/g/s9_tma_new python bench.py --workload stencil9 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g/ncu_f.log 2>&1
tail -2 gpurun_out/g/pytest.log
for f in gpurun_out/g/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
