# checkpoint: full GPU suite on 4 GPUs + every bench workload at N=1/2/4
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/r
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r/pytest.log
tail -n 3 gpurun_out/r/pytest.log
TAG=r/all NG=4 bash tools/bench_all.sh
