# session 4: TMA bulk feed of the DMMA GEMM tiles -- GEMM numerics, large-path parity, A/B
# against the cp.async-only build (libqtt_notma.so = -DQTT_GEMM_TMA=0)
set -x
O=gpurun_out/s4a; mkdir -p $O; rm -f gpurun_out/ab.txt
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -s > $O/pytest_gemm.log 2>&1; echo gemm_rc=$?
tail -3 $O/pytest_gemm.log
for w in cfg3 cfg4 cfg2; do bash scripts/ab_large.sh $w base notma bkt base notma bkt; done
cp gpurun_out/ab.txt $O/ab_tma.txt; cat $O/ab_tma.txt
timeout 2400 python -m pytest tests/test_gpu_large.py tests/test_gpu_shard.py tests/test_gpu_f32.py -q -p no:cacheprovider --timeout 600 > $O/pytest_large.log 2>&1; echo large_rc=$?
tail -3 $O/pytest_large.log
QTT_LIB=paper_2602_20226_b200/lib/libqtt_bkt.so timeout 2400 python -m pytest tests/test_gpu_large.py tests/test_gpu_shard.py -q -p no:cacheprovider --timeout 600 > $O/pytest_large_bkt.log 2>&1; echo large_bkt_rc=$?
tail -3 $O/pytest_large_bkt.log
