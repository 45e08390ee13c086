# batched corrected-reciprocal divisions: parity, standalone designs, bench A/B
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/f
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo tools/stencil_tma_tune.cu -o tools/stencil_tma_tune -lcuda
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "stencil or config2 or tma" > gpurun_out/f/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f/pytest.log
HDA_DIV=1 timeout 600 ./tools/stencil_tma_tune 20 14 > gpurun_out/f/tune14_div1.txt 2>&1
HDA_DIV=0 timeout 300 ./tools/stencil_tma_tune 20 13 > gpurun_out/f/tune13_div0.txt 2>&1
for d in 0 1 0 1; do HDA_DIV=$d timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/f/s9_div$d.$RANDOM.json 2>/dev/null; done
for d in 0 1 0 1; do HDA_DIV=$d timeout 300 python bench.py --workload stencil7 --no-cpu-baseline --no-e2e > gpurun_out/f/s7_div$d.$RANDOM.json 2>/dev/null; done
HDA_TMA=0 timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/f/s9_tma0_div1.json 2>/dev/null
tail -3 gpurun_out/f/pytest.log
cat gpurun_out/f/tune14_div1.txt gpurun_out/f/tune13_div0.txt
for f in gpurun_out/f/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
