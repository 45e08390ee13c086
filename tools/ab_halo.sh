#!/bin/bash
# A/B the 2-D halo launch shapes (HDA_HALO_MODE) at N=2 and N=4 (torchrun, one rank per GPU).
set -u
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29611"
TAG=${TAG:-ab}
if [ -z "${SKIP_N1:-}" ]; then
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_j_n1.json 2> gpurun_out/${TAG}_j_n1.err
  timeout 300 python bench.py --no-cpu-baseline --workload stencil9 > gpurun_out/${TAG}_s9_n1.json 2> gpurun_out/${TAG}_s9_n1.err
fi
for mode in ${MODES:-0 1}; do
  for n in 2 4; do
    HDA_HALO_MODE=$mode timeout 300 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline ${EXTRA:-} \
      > gpurun_out/${TAG}_j_m${mode}_n$n.json 2> gpurun_out/${TAG}_j_m${mode}_n$n.err
    HDA_HALO_MODE=$mode timeout 300 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline \
      --workload stencil9 > gpurun_out/${TAG}_s9_m${mode}_n$n.json 2> gpurun_out/${TAG}_s9_m${mode}_n$n.err
  done
done
for f in gpurun_out/${TAG}_*.json; do
  printf "%-32s " $(basename $f)
  grep '"metric"' $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["ms_per_step"], (d.get("roofline") or {}).get("frac"))' 2>/dev/null || echo FAIL
done
