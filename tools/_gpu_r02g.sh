python -m pytest tests/test_gpu_truncated_stats.py -m gpu -q -p no:cacheprovider -k c2 > gpurun_out/r02g_stat_c2.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02g_stat_c2.log
python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "bench exit $?" >> gpurun_out/r02g_bench.err
python tools/run_c5_full.py t0 gpurun_out/c5_t0.mps > gpurun_out/r02g_c5_t0.log 2>&1; echo "c5 exit $?" >> gpurun_out/r02g_c5_t0.log
