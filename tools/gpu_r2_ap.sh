# forced fused halo launch at 8192^2 N=4 (268 MB shares): in-kernel vs trailing signal, pull-block cap
mkdir -p gpurun_out/ap
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
b() { tag=$1; shift; timeout 600 env HDA_HALO_MODE=1 "$@" $TR --nproc-per-node 4 bench.py --gpus 4 --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/ap/$tag.json 2>/dev/null; }
b trail1 HDA_HALO_SIG_TRAIL=1
b trail1_np64 HDA_HALO_SIG_TRAIL=1 HDA_HALO_NPULL=64
b trail0_np64 HDA_HALO_SIG_TRAIL=0 HDA_HALO_NPULL=64
for f in gpurun_out/ap/*.json; do printf "%-20s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
