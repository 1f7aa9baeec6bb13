# ncu --set full of one launch of each per-member kernel: k_zipup<complex> (qft chain),
# k_variational (one sweep over 512 cfg5 members), k_zipup<double> (cfg5 window 2);
# each command first run plain (exit 0)
Q="python bench.py --workload qft --steps 1 --warmup 3 --no-cpu-baseline"
V="python bench.py --workload variational --steps 1 --warmup 3 --no-cpu-baseline"
W="python bench.py --window 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$Q > gpurun_out/plain_qft.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zipup" -s 20 -c 1 -o gpurun_out/prof_qft $Q > gpurun_out/ncu_qft.log 2>&1
$V > gpurun_out/plain_var.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_variational" -s 3 -c 1 -o gpurun_out/prof_var $V > gpurun_out/ncu_var.log 2>&1
$W > gpurun_out/plain_w2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zipup" -s 3 -c 1 -o gpurun_out/prof_w2 $W > gpurun_out/ncu_w2.log 2>&1
