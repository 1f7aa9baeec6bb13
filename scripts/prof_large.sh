# launch list (device time per kernel) of one zip-up of a large-member workload: prof_large.sh cfg3
W=${1:-cfg3}
C="python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain_$W.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_$W.csv $C > gpurun_out/ncu_$W.log 2>&1
