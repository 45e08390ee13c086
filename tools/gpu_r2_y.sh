# multi-GPU parity after the in-kernel halo signal; N=8-sized share A/B
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/y
timeout 2400 python -m pytest tests/test_gpu_spmd.py tests/test_gpu_parity.py tests/test_gpu_fullscale.py -q -m gpu -p no:cacheprovider -x -k "not gemm and not 2mm" > gpurun_out/y/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/y/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for t in 0 1; do
HDA_HALO_SIG_TRAIL=$t timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/y/j5792_trail$t.json 2>/dev/null
done
tail -n 3 gpurun_out/y/pytest.log
for f in gpurun_out/y/j*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
