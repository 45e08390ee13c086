# closing validation of the final tree on two GPUs: full GPU suite + smoke + default line
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/final7; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_n1.json 2>/dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.json 2>/dev/null
tail -n 2 $O/pytest.log; tail -n 2 $O/smoke.log
for f in $O/bench_n*.json; do tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["n_gpus"], round(d["value"],1), d["unit"], round(d["roofline"]["frac"],3), d["e2e"]["value"], d["gpu_launches"], d["clocks"]["reasons"])'; done
