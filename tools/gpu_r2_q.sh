# 2-D register-march stencils: L2 bulk prefetch distance sweep (HDA_ST_PF / HDA_ST9_PF); 3-D PF 1 vs 2
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/q
HDA_ST_PF=2 HDA_ST9_PF=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stencil or config or edge or eigen or jacobi" > gpurun_out/q/pytest.log 2>&1
for i in 1 2; do
  for p in 0 1 2 3; do HDA_ST9_PF=$p timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/q/s9_pf$p.$i.json 2>/dev/null; done
  for p in 0 1 2; do HDA_ST_PF=$p timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/q/j_pf$p.$i.json 2>/dev/null; done
  for p in 1 2; do HDA_S7_PF=$p timeout 300 python bench.py --workload stencil7 --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/q/s7_pf$p.$i.json 2>/dev/null; done
done
tail -n 2 gpurun_out/q/pytest.log
for f in gpurun_out/q/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
