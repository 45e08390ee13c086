# 9-point tile-height rule (32 rows when >= 10 waves): parity + N=1/2/4 bench
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/av
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py -q -p no:cacheprovider -k "stencil or config or edge or eigen or block or 9" > gpurun_out/av/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/av/pytest.log
timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/av/s9_n1.json 2>/dev/null
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/av/s9_n2.json 2>/dev/null
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/av/s9_n4.json 2>/dev/null
tail -n 2 gpurun_out/av/pytest.log
for f in gpurun_out/av/*.json; do printf "%-16s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
