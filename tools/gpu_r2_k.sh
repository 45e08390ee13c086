# cost of per-segment passes on an ungated 16384^2 GEMM (fp32 C), N=1
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/k
for i in 1 2; do for s in 0 2 4; do
HDA_DEBUG_GEMM_SEGS=$s timeout 300 python bench.py --workload gemm --no-cpu-baseline --no-e2e > gpurun_out/k/gemm_seg$s.$i.json 2>/dev/null
done; done
for f in gpurun_out/k/*.json; do printf "%-26s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), round(d.get("ms_per_step",0),4), r.get("frac"), d.get("parity"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
