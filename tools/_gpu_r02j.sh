# cluster Jacobi: parity tests, A/B timing, headline bench (no regression)
timeout 1200 python -m pytest tests/test_gpu_cluster.py -q -x -p no:cacheprovider > gpurun_out/r02j_cluster_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02j_cluster_tests.log
timeout 900 python tools/time_cluster.py 25 > gpurun_out/r02j_time_cluster.log 2>&1; echo "exit $?" >> gpurun_out/r02j_time_cluster.log
python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench exit $?" >> gpurun_out/r02j_bench.err
