set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --members-per-gpu 296"
$B > gpurun_out/plain_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
$P > gpurun_out/plain_p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/prof_sweep $P > gpurun_out/ncu_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_orth -s 2 -c 1 -o gpurun_out/prof_orth $P > gpurun_out/ncu_orth.log 2>&1
ls -la gpurun_out
