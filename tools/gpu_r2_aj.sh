# split product, one launch per source as its rows land: parity + 2MM ROW at N=2 / N=4
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/aj
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rA -k "gated_allgather and (2-2 or 2-4)" 2>&1 | grep -E "PASS|FAIL|passed|failed|Error|MISMATCH" > gpurun_out/aj/pytest.log
for i in 1 2; do
  timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/aj/2mm_row_n4.$i.json 2>/dev/null
  timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/aj/2mm_row_n2.$i.json 2>/dev/null
done
cat gpurun_out/aj/pytest.log
for f in gpurun_out/aj/2mm*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
