# 9-point: cached row edges / pair sums (ST9_EDGE_CACHE) x rows per group (ST9_GROUP) x prefetch distance
mkdir -p gpurun_out/ae
run() {  # tag flags pf
  HDA_NVCC_FLAGS="$2" python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
  for i in 1 2; do
    HDA_ST9_PF=$3 HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/ae/s9_$1.$i.json 2>/dev/null
  done
  HDA_ST9_PF=$3 HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/ae/s9_$1.def.json 2>/dev/null
}
run nocache_g4 "-DST9_EDGE_CACHE=0" 1
run cache_g4 "-DST9_GROUP=4" 1
run cache_g3 "-DST9_GROUP=3" 1
run cache_g2_pf1 "-DST9_GROUP=2" 1
run cache_g2_pf2 "-DST9_GROUP=2" 2
run cache_g2_pf3 "-DST9_GROUP=2" 3
python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
HDA_AUTOBUILD=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stencil or config or edge or eigen" > gpurun_out/ae/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ae/pytest.log
tail -n 2 gpurun_out/ae/pytest.log
for f in gpurun_out/ae/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
