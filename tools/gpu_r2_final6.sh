# driver-like closing check on one GPU: build, GPU suite, smoke, default bench line, reference arm
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/final6; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_n1.json 2>/dev/null
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/reference_n1.json 2>/dev/null
tail -n 2 $O/pytest.log; tail -n 2 $O/smoke.log
tail -1 $O/bench_n1.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"], d["unit"], d["roofline"]["frac"], d["e2e"]["value"], d["cpu_baseline"]["value"], d["gpu_launches"], d["clocks"])'
tail -1 $O/reference_n1.json | cut -c1-300
