# cluster-Jacobi debug switches; Gram screen (DMMA) of the late Jacobi sweeps + small-problem engine: parity, then A/B
timeout 900 python tools/dbg_cluster129.py > gpurun_out/r02m_dbg_cluster.log 2>&1; echo "exit $?" >> gpurun_out/r02m_dbg_cluster.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_small_engine.py tests/test_gpu_robustness.py -q -p no:cacheprovider > gpurun_out/r02m_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02m_pytest.log
for gs in 1 0; do
  TB_GRAM_SCREEN=$gs timeout 600 python tools/time_prefix.py 32 64 4 5 200 2.0 148 30 > gpurun_out/r02m_prefix30_screen$gs.log 2>&1
done
TB_GRAM_SCREEN=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02m_bench_screen1.json 2> gpurun_out/r02m_bench_screen1.err
TB_GRAM_SCREEN=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02m_bench_screen0.json 2> gpurun_out/r02m_bench_screen0.err
timeout 900 python tools/ab_small_engine.py > gpurun_out/r02m_ab_small_engine.log 2>&1; echo "exit $?" >> gpurun_out/r02m_ab_small_engine.log
