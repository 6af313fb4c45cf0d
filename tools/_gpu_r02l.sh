# cluster TMA race fix: hammer the 129x129 case; full GPU suite; whole-config C5 / C4 chi=128 runs
timeout 900 python tools/dbg_cluster129.py > gpurun_out/r02l_dbg_cluster.log 2>&1; echo "exit $?" >> gpurun_out/r02l_dbg_cluster.log
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02l_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02l_pytest.log
timeout 1500 python tools/run_c5_full.py t0 gpurun_out/c5_t0.mps > gpurun_out/r02l_c5_t0.log 2>&1; echo "exit $?" >> gpurun_out/r02l_c5_t0.log
timeout 1500 python tools/run_c5_full.py tepai gpurun_out/c5_t0.mps 148 > gpurun_out/r02l_c5_tepai.log 2>&1; echo "exit $?" >> gpurun_out/r02l_c5_tepai.log
timeout 2400 python tools/run_c4_full.py 128 148 > gpurun_out/r02l_c4_chi128.log 2>&1; echo "exit $?" >> gpurun_out/r02l_c4_chi128.log
