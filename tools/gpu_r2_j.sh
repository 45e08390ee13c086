# 2MM ROW timelines (trace) gate 0 / 1 at N=2, CE copy under GEMM load
python -m paper_1809_05657_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/j
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29631 --nproc-per-node 2"
timeout 300 python tools/ce_contention.py > gpurun_out/j/ce.txt 2>&1; cat gpurun_out/j/ce.txt; exit 0
for g in 0 1; do
HDA_GEMM_GATE=$g timeout 600 $TR bench.py --gpus 2 --workload 2mm --part row --steps 6 --warmup 3 --trace 3 --no-cpu-baseline --no-e2e > gpurun_out/j/2mm_gate$g.json 2>/dev/null
for r in 0 1; do mv gpurun_out/trace_2mm_n2_r$r.json gpurun_out/j/trace_gate${g}_r$r.json; done
done
cat gpurun_out/j/ce.txt
