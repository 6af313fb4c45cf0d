# after the qrcp_mgs pivot-candidate double buffering: determinism (small engine, two CTAs per SM), full GPU suite, bench
for i in 1 2 3; do
  timeout 600 python tools/check_determinism.py > gpurun_out/r02r_det_$i.log 2>&1; echo "exit $?" >> gpurun_out/r02r_det_$i.log
done
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02r_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02r_pytest.log
python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench exit $?" >> gpurun_out/r02r_bench.err
timeout 900 python tools/ab_small_engine.py > gpurun_out/r02r_ab_small_engine.log 2>&1; echo "exit $?" >> gpurun_out/r02r_ab_small_engine.log
