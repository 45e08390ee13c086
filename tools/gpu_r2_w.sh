# N=8-sized shares on 4 GPUs (5792^2 Jacobi = 134 MB per GPU, the L2-flush mode): split vs fused halo
mkdir -p gpurun_out/w
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for m in -2 0 1; do
HDA_HALO_MODE=$m timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/w/j5792_m$m.json 2>/dev/null
done
HDA_HALO_MODE=-2 timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 40 --trace 6 --no-cpu-baseline --no-e2e > gpurun_out/w/j5792_tr.json 2>/dev/null
for r in 0 1 2 3; do mv gpurun_out/trace_jacobi2d_n4_r$r.json gpurun_out/w/; done
timeout 600 python bench.py --size 2896 --steps 40 --no-cpu-baseline --no-e2e > gpurun_out/w/j2896_n1.json 2>/dev/null
for f in gpurun_out/w/j*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["config"]["l2"][:20])'; done
