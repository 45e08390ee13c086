# 3-D 7-point: bulk L2 prefetch distance sweep (HDA_S7_PF)
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/p
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stencil7" > gpurun_out/p/pytest.log 2>&1
HDA_S7_PF=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stencil7 or edge" >> gpurun_out/p/pytest.log 2>&1
for i in 1 2; do for p in 0 2 3 4 6; do
  HDA_S7_PF=$p timeout 300 python bench.py --workload stencil7 --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/p/s7_pf$p.$i.json 2>/dev/null
done; done
tail -n 2 gpurun_out/p/pytest.log
for f in gpurun_out/p/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
