python -m pytest tests -m gpu -q -p no:cacheprovider -k "not c3" > gpurun_out/r02c_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02c_pytest_gpu.log
python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench exit $?" >> gpurun_out/r02c_bench.err
