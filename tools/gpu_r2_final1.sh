# round-2 measurement, one GPU: N=1 bench lines, reference arm, smoke, launch list, ncu --set full of each
# workload's dominant kernel
python -m paper_1809_05657_b200.build > /dev/null 2>&1
O=gpurun_out/final1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/default_n1.json 2> $O/default_n1.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/default_n1_driver.json 2>/dev/null
timeout 600 python bench.py --impl reference > $O/reference_n1.json 2>/dev/null
for w in stencil9 stencil7 repartition gemm 2mm; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/${w}_n1.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
cap() {  # name regex workload-args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 8 -c 1 -o $O/$1 \
    python bench.py $3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$1.log 2>&1
}
cap jacobi stencil2d_kernel ""
cap stencil9 stencil2d_kernel "--workload stencil9"
cap stencil7 stencil7_kernel "--workload stencil7"
cap gemm gemm2_kernel "--workload gemm"
cat $O/smoke.log | tail -2
for f in $O/*.json; do printf "%-28s " $(basename $f); grep '"metric"' $f | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0),4), r.get("frac"), (d.get("e2e") or {}).get("value"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
ls $O
