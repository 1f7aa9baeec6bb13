# session 3: A/B of the per-CTA site-matrix scratch (base) against per-member slots (old), the
# small-path GPU tests, DRAM bytes of k_sweep per variant
O=gpurun_out/s3a; mkdir -p $O
bash scripts/ab.sh base old base old > /dev/null 2>&1; cp gpurun_out/ab.txt $O/ab.txt
timeout 900 python -m pytest tests/test_gpu_zipup.py tests/test_gpu_large.py tests/test_gpu_exact.py -m gpu -q -p no:cacheprovider -k "not full_oracle" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
for v in base old; do
  if [ $v = base ]; then lib=paper_2602_20226_b200/lib/libqtt.so; else lib=paper_2602_20226_b200/lib/libqtt_old.so; fi
  QTT_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_sweep" -s 1 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$v.csv 2>&1; echo ncu_$v=$?
done
