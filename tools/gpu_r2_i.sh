# gated product with per-segment passes: parity at 2 GPUs, 2MM ROW A/B at N=2
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/i
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631 --nproc-per-node 2"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm or 2mm" > gpurun_out/i/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i/pytest.log
timeout 900 python -m pytest tests/test_gpu_spmd.py -x -q -p no:cacheprovider -k "two and plain" > gpurun_out/i/pytest_spmd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i/pytest_spmd.log
for i in 1 2; do
HDA_GEMM_GATE=0 timeout 600 $TR bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/i/2mm_row_gate0.$i.json 2>/dev/null
HDA_GEMM_GATE=1 HDA_GATE_PASSES=1 timeout 600 $TR bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/i/2mm_row_pass1.$i.json 2>/dev/null
HDA_GEMM_GATE=1 HDA_GATE_PASSES=0 timeout 600 $TR bench.py --gpus 2 --workload 2mm --part row --no-cpu-baseline --no-e2e > gpurun_out/i/2mm_row_pass0.$i.json 2>/dev/null
done
timeout 600 $TR bench.py --gpus 2 --workload 2mm --part col --no-cpu-baseline --no-e2e > gpurun_out/i/2mm_col.json 2>/dev/null
tail -n 3 gpurun_out/i/pytest.log gpurun_out/i/pytest_spmd.log
for f in gpurun_out/i/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
