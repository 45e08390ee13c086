#!/bin/bash
# Every bench workload at N=1 and N=NG (torchrun), plus the reference arm and the
# default line; JSON lines into gpurun_out/${TAG}_*.json.
set -u
mkdir -p gpurun_out
TAG=${TAG:-all}
NG=${NG:-4}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29621"
timeout 900 python bench.py > gpurun_out/${TAG}_default_n1.json 2> gpurun_out/${TAG}_default_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_reference_n1.json 2>/dev/null
for w in stencil9 stencil7 repartition gemm; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${TAG}_${w}_n1.json 2>/dev/null
done
for n in 2 $NG; do
  for w in jacobi2d stencil9 stencil7 repartition gemm; do
    timeout 600 $TR --nproc-per-node $n bench.py --gpus $n --workload $w --no-cpu-baseline \
      > gpurun_out/${TAG}_${w}_n$n.json 2>/dev/null
  done
done
timeout 600 $TR --nproc-per-node $NG bench.py --gpus $NG --size 5792 --no-cpu-baseline > gpurun_out/${TAG}_jacobi5792_flush_n$NG.json 2>/dev/null
timeout 600 $TR --nproc-per-node $NG bench.py --gpus $NG --impl reference > gpurun_out/${TAG}_reference_n$NG.json 2>/dev/null
for f in gpurun_out/${TAG}_*.json; do
  printf "%-40s " $(basename $f)
  grep '"metric"\|"unavailable"' $f | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), "ms/step", round(d.get("ms_per_step",0),4), "frac", r.get("frac"), "e2e", (d.get("e2e") or {}).get("value"), "L", d.get("gpu_launches"), d.get("config",{}).get("l2",""))' 2>/dev/null || echo FAIL
done
