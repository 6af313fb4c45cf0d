python -m pytest tests/test_gpu_truncated_stats.py -q -p no:cacheprovider > gpurun_out/r02t_pytest_stats.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02t_pytest_stats.log
bash tools/_gpu_r02s.sh
