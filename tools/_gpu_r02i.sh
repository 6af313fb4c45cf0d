# round-2 re-entry: sanity of the restored tree, then the whole-config C5 / C4 chi=128 runs
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02i_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02i_pytest.log
python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "bench exit $?" >> gpurun_out/r02i_bench.err
timeout 1800 python tools/run_c5_full.py t0 gpurun_out/c5_t0.mps > gpurun_out/r02i_c5_t0.log 2>&1; echo "exit $?" >> gpurun_out/r02i_c5_t0.log
timeout 1500 python tools/run_c5_full.py tepai gpurun_out/c5_t0.mps 148 > gpurun_out/r02i_c5_tepai.log 2>&1; echo "exit $?" >> gpurun_out/r02i_c5_tepai.log
timeout 1500 python tools/run_c4_full.py 128 148 --ensemble-only > gpurun_out/r02i_c4_chi128.log 2>&1; echo "exit $?" >> gpurun_out/r02i_c4_chi128.log
