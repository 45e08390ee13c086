# forced fused halo launch at 8192^2 N=4: prefetch off / one-wave off
mkdir -p gpurun_out/aq
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
b() { tag=$1; shift; timeout 600 env HDA_HALO_MODE=1 "$@" $TR --nproc-per-node 4 bench.py --gpus 4 --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/aq/$tag.json 2>/dev/null; }
b pf0 HDA_ST_PF=0
b pf0_ow0 HDA_ST_PF=0 HDA_ONE_WAVE=0
b ow0 HDA_ONE_WAVE=0
b pdl0 HDA_PDL=0
for f in gpurun_out/aq/*.json; do printf "%-20s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
