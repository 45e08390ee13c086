# N=8-sized Jacobi share on one GPU (2896^2 = 134 MB per step, flush mode): layout / prefetch sweep
mkdir -p gpurun_out/aa
b() { timeout 300 env "$@" python bench.py --size 2896 --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/aa/$(echo "$@" | tr ' =' '_-').json 2>/dev/null; }
b HDA_ST_PF=1
b HDA_ST_PF=2
b HDA_ST_PF=3
b HDA_ST_PF=0
b HDA_TAIL_ROWS=0
b HDA_TAIL_ROWS=0 HDA_ST_PF=2
b HDA_TAIL_ROWS=8
b HDA_PDL=0
b HDA_TMA=2
for f in gpurun_out/aa/*.json; do printf "%-34s " $(basename $f); tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d.get("roofline") or {}; print(round(d.get("value",0),1), d.get("unit"), d["steps"], round(d.get("ms_per_step",0)*1000,2), "us", r.get("frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'; done
