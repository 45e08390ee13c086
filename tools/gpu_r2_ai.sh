# N=8-sized Jacobi shares on 4 GPUs (5792^2): fused-halo pull-block cap, one-wave layout
mkdir -p gpurun_out/ai
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
b() { tag=$1; shift; timeout 600 env "$@" $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/ai/$tag.json 2>/dev/null; }
for i in 1 2; do
b np64.$i HDA_HALO_NPULL=64
b np16.$i HDA_HALO_NPULL=16
b np4.$i HDA_HALO_NPULL=4
b ow0.$i HDA_ONE_WAVE=0
done
b depfirst0 HDA_DEP_FIRST=0
b pf0 HDA_ST_PF=0
b pf2 HDA_ST_PF=2
for f in gpurun_out/ai/*.json; do printf "%-16s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
