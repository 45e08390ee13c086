# Jacobi: TMA ring vs register march across share sizes, N=1 and N=4
mkdir -p gpurun_out/ab
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for n in 2896 4096 5792 8192; do for t in 0 2; do
  HDA_TMA=$t timeout 300 python bench.py --size $n --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/ab/n1_s${n}_tma$t.json 2>/dev/null
done; done
for t in 0 2; do for m in -2 0; do
  HDA_TMA=$t HDA_HALO_MODE=$m timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/ab/n4_s5792_tma${t}_m$m.json 2>/dev/null
  HDA_TMA=$t HDA_HALO_MODE=$m timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 8192 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/ab/n4_s8192_tma${t}_m$m.json 2>/dev/null
done; done
for t in 0 2; do
  HDA_TMA=$t timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --size 8192 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/ab/n2_s8192_tma$t.json 2>/dev/null
done
for f in gpurun_out/ab/*.json; do printf "%-28s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
