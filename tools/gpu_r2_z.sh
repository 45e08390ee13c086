# 9-point register cap (ST9_MINB 4 / 5 / 6) with div20 + prefetch, N=1
mkdir -p gpurun_out/z
run() {
  HDA_NVCC_FLAGS="$2" python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
  for i in 1 2; do
    HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/z/s9_$1.40.$i.json 2>/dev/null
  done
  HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/z/s9_$1.def.json 2>/dev/null
}
run m5 "-DST9_MINB=5"
run m4 "-DST9_MINB=4"
run m6 "-DST9_MINB=6"
HDA_ST9_PF=2 run m5pf2 "-DST9_MINB=5"
python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
for f in gpurun_out/z/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
