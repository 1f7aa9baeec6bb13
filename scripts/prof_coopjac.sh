C="python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_jacobi_coop -s 80 -c 1 -o gpurun_out/prof_coopjac $C > gpurun_out/ncu_coopjac.log 2>&1
