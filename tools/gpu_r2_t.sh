# 3-D prefetch: own rows only (pf+16) vs with halo rows, default steps, interleaved
mkdir -p gpurun_out/t
for i in 1 2; do for p in 2 18 3 19; do
  HDA_S7_PF=$p timeout 300 python bench.py --workload stencil7 --no-cpu-baseline --no-e2e > gpurun_out/t/s7_pf$p.$i.json 2>/dev/null
done; done
for f in gpurun_out/t/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
