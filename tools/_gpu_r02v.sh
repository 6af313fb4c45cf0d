# flag-driven within phase (TB_GRAM_SCREEN=3, default) vs 2: parity, A/B, determinism; truncated-regime tests in both modes
python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_small_engine.py -q -p no:cacheprovider > gpurun_out/r02v_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02v_pytest.log
for gs in 3 2; do
  TB_GRAM_SCREEN=$gs timeout 900 python tools/time_prefix.py 32 64 4 5 200 2.0 148 60 > gpurun_out/r02v_prefix60_screen$gs.log 2>&1
done
TB_GRAM_SCREEN=3 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02v_bench_screen3.json 2> gpurun_out/r02v_bench_screen3.err
TB_GRAM_SCREEN=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02v_bench_screen2.json 2> gpurun_out/r02v_bench_screen2.err
for i in 1 2; do timeout 600 python tools/check_determinism.py > gpurun_out/r02v_det_$i.log 2>&1; done
python -m pytest tests/test_gpu_truncated_stats.py -q -p no:cacheprovider > gpurun_out/r02v_pytest_stats.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02v_pytest_stats.log
