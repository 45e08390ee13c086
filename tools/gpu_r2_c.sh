python -m paper_1809_05657_b200.build
mkdir -p gpurun_out
for p in 1 0; do for t in 0 1 0 1; do HDA_PDL=$p HDA_TMA=$t python bench.py --workload stencil9 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$p tma=$t', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; done; done
