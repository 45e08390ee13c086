# 3-D: rows per thread (S3_R) and planes per block (S3_ZCH) with own-row prefetch, default steps
mkdir -p gpurun_out/u
run() {  # tag, nvcc flags, pf
  HDA_NVCC_FLAGS="$2" python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
  for i in 1 2; do
    HDA_AUTOBUILD=0 HDA_S7_PF=$3 timeout 300 python bench.py --workload stencil7 --no-cpu-baseline --no-e2e > gpurun_out/u/s7_$1.$i.json 2>/dev/null
  done
}
run r2_pf18 "-DS3_R_DEF=2" 18
run r4_pf18 "-DS3_R_DEF=4" 18
run r4_pf17 "-DS3_R_DEF=4" 17
run r2_z64_pf18 "-DS3_R_DEF=2 -DS3_ZCH_DEF=64" 18
run r1_pf18 "-DS3_R_DEF=1" 18
run r1_pf19 "-DS3_R_DEF=1" 19
run r2_pf17 "-DS3_R_DEF=2" 17
python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
for f in gpurun_out/u/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
