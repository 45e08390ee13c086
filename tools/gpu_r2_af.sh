# comm-stream pull: RAW/WAR waits in a one-CTA kernel before the copy (HDA_PULL_WAIT_KERNEL=1) vs folded
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/af
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631"
for i in 1 2; do for pw in 1 0; do
  HDA_PULL_WAIT_KERNEL=$pw timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/af/j_n4_pw$pw.$i.json 2>/dev/null
  HDA_PULL_WAIT_KERNEL=$pw timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload stencil9 --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/af/s9_n4_pw$pw.$i.json 2>/dev/null
  HDA_PULL_WAIT_KERNEL=$pw timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --workload stencil7 --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/af/s7_n4_pw$pw.$i.json 2>/dev/null
done; done
for pw in 1 0; do
  HDA_PULL_WAIT_KERNEL=$pw timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/af/j_n2_pw$pw.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_spmd.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "spmd or war or config or halo or multi or gpus" > gpurun_out/af/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/af/pytest.log
tail -n 2 gpurun_out/af/pytest.log
for f in gpurun_out/af/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
