# round 2 (session 2) evidence: full GPU suite, smoke, every bench line, reference arm, cfg5 launch
# list, ncu --set full of k_sweep and k_orth (512 members) for the traffic figures
set -x
O=gpurun_out/${R02_OUT:-r02final2}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --durations 15 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
timeout 900 python bench.py --strong --steps 5 --warmup 3 > $O/bench_cfg5_strong4096.json 2> $O/bench_cfg5_strong.err; echo strong=$?
for W in cfg1 cfg2 cfg3 cfg4; do timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > $O/bench_$W.json 2> $O/bench_$W.err; echo $W=$?; done
timeout 600 python bench.py --workload cfg3 --dtype f32 --steps 5 --warmup 3 > $O/bench_cfg3_f32.json 2> $O/bench_cfg3_f32.err; echo f32=$?
timeout 300 python bench.py --workload qft --steps 5 --warmup 3 > $O/bench_qft.json 2> $O/bench_qft.err; echo qft=$?
timeout 300 python bench.py --workload variational --steps 5 --warmup 3 > $O/bench_var1.json 2> $O/bench_var1.err; echo var1=$?
timeout 300 python bench.py --workload variational --ncores 2 --steps 5 --warmup 3 > $O/bench_var2.json 2> $O/bench_var2.err; echo var2=$?
timeout 600 python bench.py --window 2 --steps 5 --warmup 3 > $O/bench_w2.json 2> $O/bench_w2.err; echo w2=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/ref_cfg5.json 2> $O/ref_cfg5.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_cfg5.log 2>&1; echo ncu=$?
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_orth" -s 6 -c 3 -o $O/sweep_orth $P > $O/ncu_full.log 2>&1; echo ncufull=$?
ncu -i $O/sweep_orth.ncu-rep --page raw --csv > $O/sweep_orth_raw.csv 2>/dev/null
ncu -i $O/sweep_orth.ncu-rep --page source --csv --print-source cuda,sass > $O/sweep_orth_source.csv 2>/dev/null
python scripts/ncu_lines.py 60 < $O/sweep_orth_source.csv > $O/sweep_orth_lines.txt 2>/dev/null
rm -f $O/sweep_orth_source.csv
