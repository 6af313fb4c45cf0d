# flag-driven cross phase of the screened sweeps (TB_GRAM_SCREEN=2, default) vs the first screened version (1): parity, A/B
python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_small_engine.py -q -p no:cacheprovider > gpurun_out/r02u_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02u_pytest.log
for gs in 2 1; do
  TB_GRAM_SCREEN=$gs timeout 900 python tools/time_prefix.py 32 64 4 5 200 2.0 148 60 > gpurun_out/r02u_prefix60_screen$gs.log 2>&1
done
TB_GRAM_SCREEN=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02u_bench_screen2.json 2> gpurun_out/r02u_bench_screen2.err
TB_GRAM_SCREEN=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02u_bench_screen1.json 2> gpurun_out/r02u_bench_screen1.err
for i in 1 2; do timeout 600 python tools/check_determinism.py > gpurun_out/r02u_det_$i.log 2>&1; done
