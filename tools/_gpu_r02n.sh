# cluster tests with the clean-sweep criterion; small-engine tests; determinism check; Gram-screen phase profile
python -m pytest tests/test_gpu_cluster.py tests/test_gpu_small_engine.py -q -p no:cacheprovider > gpurun_out/r02n_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02n_pytest.log
timeout 900 python tools/check_determinism.py > gpurun_out/r02n_determinism.log 2>&1; echo "exit $?" >> gpurun_out/r02n_determinism.log
for gs in 1 0; do
  TB_GRAM_SCREEN=$gs timeout 900 python tools/time_prefix.py 32 64 4 5 200 2.0 148 60 > gpurun_out/r02n_prefix60_screen$gs.log 2>&1
done
