# prefetch gains vs step count (default bench steps vs short runs)
mkdir -p gpurun_out/s
for p in 0 2; do
  HDA_S7_PF=$p timeout 300 python bench.py --workload stencil7 --no-cpu-baseline --no-e2e > gpurun_out/s/s7_pf$p.def.json 2>/dev/null
  HDA_S7_PF=$p timeout 300 python bench.py --workload stencil7 --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/s/s7_pf$p.30.json 2>/dev/null
done
for p in 0 1; do
  HDA_ST9_PF=$p timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/s/s9_pf$p.def.json 2>/dev/null
  HDA_ST9_PF=$p timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/s/s9_pf$p.40.json 2>/dev/null
done
for f in gpurun_out/s/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
