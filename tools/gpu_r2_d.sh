# round 2 re-entry: full GPU suite, every N=1 workload, TMA A/B for the 2-D stencils,
# launch list + one full ncu capture of the 9-point TMA kernel
set -x
python -m paper_1809_05657_b200.build
mkdir -p gpurun_out/d
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/d/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/d/default_n1.json 2> gpurun_out/d/default_n1.err
for t in 0 1 2 0 1 2; do HDA_TMA=$t timeout 300 python bench.py --workload stencil9 --no-cpu-baseline --no-e2e > gpurun_out/d/s9_tma$t.$RANDOM.json 2>/dev/null; done
for t in 0 2 0 2; do HDA_TMA=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/d/j_tma$t.$RANDOM.json 2>/dev/null; done
for w in stencil7 repartition gemm; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/d/${w}_n1.json 2>/dev/null; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/d/launches_s9.csv python bench.py --workload stencil9 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d_tma -s 6 -c 1 -o gpurun_out/d/s9_tma python bench.py --workload stencil9 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d/ncu_f.log 2>&1
tail -3 gpurun_out/d/pytest.log
for f in gpurun_out/d/*.json; do printf "%-30s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), (d.get("e2e") or {}).get("value"), d["clocks"]["sm_mhz"])' 2>/dev/null || echo FAIL; done
