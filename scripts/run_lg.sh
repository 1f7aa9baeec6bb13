# large-path check: GPU tests of every path, then one zip-up of each large workload and the cfg5 bench
rm -f gpurun_out/ab.txt
python -m pytest tests -m gpu -q -x > gpurun_out/pt_all.log 2>&1
bash scripts/ab_large.sh cfg3 base
bash scripts/ab_large.sh cfg2 base
bash scripts/ab_large.sh cfg4 base
python bench.py > gpurun_out/bench_cfg5.log 2>&1
