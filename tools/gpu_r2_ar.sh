# fused halo launch without prefetch: the N=8-sized shares (its default use) and parity of the fused path
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/ar
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 900 python -m pytest tests/test_gpu_spmd.py -q -p no:cacheprovider -k "two_gpus and fused" > gpurun_out/ar/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ar/pytest.log
for i in 1 2; do
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/ar/j5792_n4.$i.json 2>/dev/null
done
tail -n 2 gpurun_out/ar/pytest.log
for f in gpurun_out/ar/*.json; do printf "%-20s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
