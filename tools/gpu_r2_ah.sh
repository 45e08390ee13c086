# split product as the default: parity (single process + SPMD), 2MM / GEMM bench at N=2
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/ah
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spmd.py -q -p no:cacheprovider -rA -k "gated or 2mm or gemm or spmd_two" 2>&1 | grep -E "PASS|FAIL|passed|failed|Error|MISMATCH" > gpurun_out/ah/pytest.log
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline > gpurun_out/ah/2mm_row_n2.json 2>/dev/null
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload gemm --no-cpu-baseline > gpurun_out/ah/gemm_n2.json 2>/dev/null
cat gpurun_out/ah/pytest.log
for f in gpurun_out/ah/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), (d.get("e2e") or {}).get("value"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
