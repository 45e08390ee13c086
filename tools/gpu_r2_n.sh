# 9-point with div20: register march (HDA_TMA=0) vs TMA ring (1), N=1 and N=2
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/n
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631 --nproc-per-node 2"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rA -k "div20" 2>&1 | grep -E "PASS|FAIL|passed|failed" > gpurun_out/n/pytest.log
for i in 1 2 3; do for t in 0 1; do
  HDA_TMA=$t timeout 300 python bench.py --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/n/s9_n1_tma$t.$i.json 2>/dev/null
done; done
for i in 1 2; do for t in 0 1; do
  HDA_TMA=$t timeout 300 $TR bench.py --gpus 2 --workload stencil9 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/n/s9_n2_tma$t.$i.json 2>/dev/null
done; done
cat gpurun_out/n/pytest.log
for f in gpurun_out/n/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
