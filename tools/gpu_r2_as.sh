# 2-D register march: rows per 16-row tile (ST_ROWS) 16 / 32 / 64 with the L2 prefetch, N=1
mkdir -p gpurun_out/as
run() {
  HDA_NVCC_FLAGS="$2" python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
  for i in 1 2; do
    HDA_AUTOBUILD=0 timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/as/s9_$1.$i.json 2>/dev/null
    HDA_AUTOBUILD=0 timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/as/j_$1.$i.json 2>/dev/null
  done
}
run r16 "-DST_ROWS_DEF=16"
run r32 "-DST_ROWS_DEF=32"
run r64 "-DST_ROWS_DEF=64"
python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
for f in gpurun_out/as/*.json; do printf "%-16s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
