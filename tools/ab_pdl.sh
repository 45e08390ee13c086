#!/bin/bash
# PDL on/off x halo mode at N=1 (8192^2 and 4096^2), N=2, N=4 (torchrun).
set -u
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29613"
TAG=${TAG:-pdl}
NG=${NG:-4}
for pdl in 1 0; do
  HDA_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_p${pdl}_j_n1.json 2>/dev/null
  HDA_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-e2e --n 4096 > gpurun_out/${TAG}_p${pdl}_j4096_n1.json 2>/dev/null
  for mode in 0 1; do
    for n in 2 $NG; do
      [ $n -gt 2 ] || [ $NG -ge 2 ] || continue
      HDA_PDL=$pdl HDA_HALO_MODE=$mode timeout 300 $TR --nproc-per-node $n bench.py --gpus $n --no-cpu-baseline --no-e2e \
        > gpurun_out/${TAG}_p${pdl}_j_m${mode}_n$n.json 2>/dev/null
    done
  done
done
for f in gpurun_out/${TAG}_*.json; do
  printf "%-32s " $(basename $f)
  grep '"metric"' $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us", (d.get("roofline") or {}).get("frac"))' 2>/dev/null || echo FAIL
done
