# round-end evidence: plain bench (512 members) then ncu --set full of one k_sweep and one
# k_orth launch of the same command, plus the launch list (gpu__time_duration per launch)
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_final.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_orth" -s 4 -c 2 -o gpurun_out/prof_final $B > gpurun_out/ncu_final.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch_final.log 2>&1
