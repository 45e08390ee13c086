#!/bin/bash
# ad-hoc A/B: runs `bench.py` at N=$N under each "VAR=val ..." setting in $CASES (separated by ';')
set -u
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29617"
TAG=${TAG:-misc}
IFS=';' read -ra CS <<< "$CASES"
i=0
for c in "${CS[@]}"; do
  if [ "${N:-1}" -gt 1 ]; then
    env $c timeout 300 $TR --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --no-e2e ${EXTRA:-} > gpurun_out/${TAG}_$i.json 2>/dev/null
  else
    env $c timeout 300 python bench.py --no-cpu-baseline --no-e2e ${EXTRA:-} > gpurun_out/${TAG}_$i.json 2>/dev/null
  fi
  printf "%-50s " "$c"
  grep '"metric"' gpurun_out/${TAG}_$i.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us", (d.get("roofline") or {}).get("frac"))' 2>/dev/null || echo FAIL
  i=$((i+1))
done
