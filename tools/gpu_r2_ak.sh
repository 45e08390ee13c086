# 9-point BLOCK N=4 and Jacobi N=4 step timelines (trace), exchange GB/s with the transfer-only timer
mkdir -p gpurun_out/ak
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload stencil9 --steps 60 --trace 4 --no-cpu-baseline --no-e2e > gpurun_out/ak/s9_n4.json 2>/dev/null
for r in 0 1 2 3; do mv gpurun_out/trace_stencil9_n4_r$r.json gpurun_out/ak/; done
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/ak/j_n4.json 2>/dev/null
for f in gpurun_out/ak/*.json; do case $f in *trace*) continue;; esac; printf "%-16s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d.get("exchange"), d["clocks"]["sm_mhz"])'; done
