# 9-point 32-row tiles for wide boxes only: N=4 / N=2 (A/B vs 16-row tiles via -DST9_ROWS=16)
mkdir -p gpurun_out/au
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for v in 32 16; do
  HDA_NVCC_FLAGS="-DST9_ROWS=$v" python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
  HDA_AUTOBUILD=0 timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/au/s9_n4_r$v.json 2>/dev/null
  HDA_AUTOBUILD=0 timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/au/s9_n2_r$v.json 2>/dev/null
done
python -m paper_1809_05657_b200.build --force > /dev/null 2>&1
for f in gpurun_out/au/*.json; do printf "%-16s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
