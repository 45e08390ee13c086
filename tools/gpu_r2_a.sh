set -x
python -m paper_1809_05657_b200.build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_n1_$i.json 2> gpurun_out/b_n1_$i.err; done
for i in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_n2_$i.json 2> gpurun_out/b_n2_$i.err; done
tail -3 gpurun_out/pytest.log
