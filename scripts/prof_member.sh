# ncu --set full of one per-member kernel launch each: k_zipup<complex> (qft chain) and
# k_variational (one sweep over 512 cfg5 members); each command first run plain (exit 0)
Q="python bench.py --workload qft --steps 1 --warmup 3 --no-cpu-baseline"
V="python bench.py --workload variational --steps 1 --warmup 3 --no-cpu-baseline --members-per-gpu 512"
$Q > gpurun_out/plain_qft.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zipup" -s 20 -c 1 -o gpurun_out/prof_qft $Q > gpurun_out/ncu_qft.log 2>&1
$V > gpurun_out/plain_var.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_variational" -s 3 -c 1 -o gpurun_out/prof_var $V > gpurun_out/ncu_var.log 2>&1
