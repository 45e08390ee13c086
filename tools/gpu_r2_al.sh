# after factoring the split product into split_product(): gated/split parity at 2 GPUs, SPMD split, 2MM N=2
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/al
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spmd.py -q -p no:cacheprovider -rA -k "gated_allgather and (2-2 or 0-2) or split_product or 2mm" 2>&1 | grep -E "PASS|FAIL|passed|failed|Error|MISMATCH" > gpurun_out/al/pytest.log
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/al/2mm_row_n2.json 2>/dev/null
cat gpurun_out/al/pytest.log
tail -1 gpurun_out/al/2mm_row_n2.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["unit"], round(d["ms_per_step"],4), d.get("parity"), d["gpu_launches"])'
