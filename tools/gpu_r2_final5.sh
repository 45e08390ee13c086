# round-2 closing measurement on four GPUs: full GPU suite, smoke, every workload at N=1/2/4
python -m paper_1809_05657_b200.build > /dev/null 2>&1
O=gpurun_out/final5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29621"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/default_n1_driver.json 2>/dev/null
timeout 900 python bench.py > $O/default_n1.json 2>/dev/null
for w in stencil9 stencil7 gemm; do timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/${w}_n1.json 2>/dev/null; done
for n in 2 4; do
  for w in jacobi2d stencil9 stencil7 repartition gemm; do
    timeout 600 $TR --nproc-per-node $n bench.py --gpus $n --workload $w --no-cpu-baseline > $O/${w}_n$n.json 2>/dev/null
  done
  for p in row col; do
    timeout 600 $TR --nproc-per-node $n bench.py --gpus $n --workload 2mm --part $p --no-cpu-baseline > $O/2mm_${p}_n$n.json 2>/dev/null
  done
done
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --size 5792 --no-cpu-baseline > $O/jacobi5792_flush_n4.json 2>/dev/null
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --impl reference --steps 20 --warmup 5 > $O/reference_n4.json 2>/dev/null
tail -n 2 $O/smoke.log; tail -n 3 $O/pytest.log
for f in $O/*.json; do printf "%-28s " $(basename $f); grep '"metric"\|"unavailable"' $f | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; x=d.get("exchange") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), x.get("GBps_per_gpu"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))' 2>/dev/null || echo FAIL; done
