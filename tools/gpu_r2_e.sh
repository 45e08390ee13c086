# 9-point / 3-D gap diagnosis: kernel vs array size, standalone designs, copy ceiling
python -m paper_1809_05657_b200.build
mkdir -p gpurun_out/e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo tools/stencil_tma_tune.cu -o tools/stencil_tma_tune -lcuda
python tools/copy_sweep.py > gpurun_out/e/copy.txt 2>&1
timeout 300 python bench.py --size 16384 --no-cpu-baseline --no-e2e > gpurun_out/e/j16384.json 2>/dev/null
timeout 300 python bench.py --workload stencil9 --size 8192 --no-cpu-baseline --no-e2e > gpurun_out/e/s9_8192.json 2>/dev/null
HDA_TMA=0 timeout 300 python bench.py --workload stencil9 --size 8192 --no-cpu-baseline --no-e2e > gpurun_out/e/s9_8192_t0.json 2>/dev/null
timeout 600 ./tools/stencil_tma_tune 20 7 > gpurun_out/e/tune7.txt 2>&1
timeout 600 ./tools/stencil_tma_tune 20 4 > gpurun_out/e/tune4.txt 2>&1
cat gpurun_out/e/copy.txt gpurun_out/e/tune7.txt gpurun_out/e/tune4.txt
for f in gpurun_out/e/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"])'; done
