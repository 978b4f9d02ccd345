B="python bench.py --code eg6 --p 64 --ebn0 4.0 --frames 2048 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plainC.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/prof_C $B > gpurun_out/ncuC.log 2>&1; echo ncu rc=$?
