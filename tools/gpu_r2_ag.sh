# split gated product (HDA_GEMM_GATE=2): parity, 2MM ROW A/B at N=2 and N=4
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/ag
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rA -k "gated" 2>&1 | grep -E "PASS|FAIL|passed|failed|Error|MISMATCH" > gpurun_out/ag/pytest.log
for i in 1 2; do for g in 0 2; do
  HDA_GEMM_GATE=$g timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/ag/2mm_row_n2_g$g.$i.json 2>/dev/null
  HDA_GEMM_GATE=$g timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/ag/2mm_row_n4_g$g.$i.json 2>/dev/null
done; done
HDA_GEMM_GATE=2 timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload 2mm --part row --steps 6 --warmup 3 --trace 3 --no-cpu-baseline --no-e2e > gpurun_out/ag/tr.json 2>/dev/null
for r in 0 1; do mv gpurun_out/trace_2mm_n2_r$r.json gpurun_out/ag/trace_g2_r$r.json; done
cat gpurun_out/ag/pytest.log
for f in gpurun_out/ag/2mm*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
