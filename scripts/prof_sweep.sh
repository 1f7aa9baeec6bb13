# ncu --set full of one k_sweep launch (296 members) after a plain run of the same command
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --members-per-gpu 296"
$P > gpurun_out/plain_p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_sweep} -s 1 -c 1 -o gpurun_out/${PROF_NAME:-prof_sweep} $P > gpurun_out/ncu_sweep.log 2>&1
