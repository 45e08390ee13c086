# ncu --set full of the 9-point kernel with 32-row tiles (the N=1 default since the tile-height rule)
O=gpurun_out/aw; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d_kernel -s 8 -c 1 -o $O/stencil9 \
  python bench.py --workload stencil9 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
tail -2 $O/ncu.log
