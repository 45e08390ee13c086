# Jacobi N=4 / N=2 step timelines (trace), default halo mode
mkdir -p gpurun_out/v
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for n in 4 2; do
timeout 600 $TR --nproc-per-node $n bench.py --gpus $n --steps 40 --warmup 5 --trace 6 --no-cpu-baseline --no-e2e > gpurun_out/v/j_n$n.json 2>gpurun_out/v/j_n$n.err
for r in $(seq 0 $((n-1))); do mv gpurun_out/trace_jacobi2d_n${n}_r$r.json gpurun_out/v/; done
done
HDA_HALO_MODE=0 timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --steps 40 --warmup 5 --trace 6 --no-cpu-baseline --no-e2e > gpurun_out/v/j_n4_m0.json 2>/dev/null
for r in 0 1 2 3; do mv gpurun_out/trace_jacobi2d_n4_r$r.json gpurun_out/v/m0_trace_jacobi2d_n4_r$r.json; done
for f in gpurun_out/v/j_*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("tracker"))'; done
