# N=8-sized shares on 4 GPUs: in-kernel PROD signal (HDA_SIG_KERNEL=0) vs trailing signal launch
mkdir -p gpurun_out/x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for i in 1 2; do for sk in 1 0; do
HDA_SIG_KERNEL=$sk timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/x/j5792_sk$sk.$i.json 2>/dev/null
HDA_SIG_KERNEL=$sk timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/x/j8192_sk$sk.$i.json 2>/dev/null
done; done
for f in gpurun_out/x/j*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
