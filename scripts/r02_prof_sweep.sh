# ncu --set full (with source) of one k_sweep launch (148 members) after a plain run; source-line table
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --members-per-gpu 148"
$P > gpurun_out/plain_p.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o gpurun_out/${PROF_NAME:-prof_sweep} $P > gpurun_out/ncu_sweep.log 2>&1
ncu -i gpurun_out/${PROF_NAME:-prof_sweep}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${PROF_NAME:-prof_sweep}_source.csv 2>/dev/null
python scripts/ncu_lines.py 60 < gpurun_out/${PROF_NAME:-prof_sweep}_source.csv > gpurun_out/${PROF_NAME:-prof_sweep}_lines.txt
ncu -i gpurun_out/${PROF_NAME:-prof_sweep}.ncu-rep --page raw --csv > gpurun_out/${PROF_NAME:-prof_sweep}_raw.csv 2>/dev/null
