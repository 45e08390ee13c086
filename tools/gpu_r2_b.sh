set -x
python -m paper_1809_05657_b200.build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "stencil or config2 or tma" > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.log
for t in 0 1 0 1; do HDA_TMA=$t python bench.py --workload stencil9 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b9_tma$t.$RANDOM.json 2>/dev/null; done
for t in 0 2 0 2; do HDA_TMA=$t python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bj_tma$t.$RANDOM.json 2>/dev/null; done
tail -3 gpurun_out/pytest_b.log
