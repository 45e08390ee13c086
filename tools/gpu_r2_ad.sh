# SPMD at 8 ranks over 4 GPUs (functional check of the N=8 protocol)
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/ad
timeout 900 python -m pytest tests/test_gpu_spmd.py -q -p no:cacheprovider -rA -k "eight or four" > gpurun_out/ad/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ad/pytest.log
tail -n 30 gpurun_out/ad/pytest.log
