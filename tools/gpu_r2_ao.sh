# Jacobi 8192^2 at N=2/N=4: split streams (default for >= 200 MB shares) vs the fused halo launch after round 2's fused-launch changes
mkdir -p gpurun_out/ao
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for i in 1 2; do for m in -2 1; do
  HDA_HALO_MODE=$m timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/ao/j_n4_m$m.$i.json 2>/dev/null
  HDA_HALO_MODE=$m timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/ao/j_n2_m$m.$i.json 2>/dev/null
done; done
for f in gpurun_out/ao/*.json; do printf "%-20s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
