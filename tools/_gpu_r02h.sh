python tools/run_c5_full.py tepai data/c5_t0.mps 148 > gpurun_out/r02h_c5_tepai.log 2>&1; echo "exit $?" >> gpurun_out/r02h_c5_tepai.log
python tools/run_c4_full.py 128 148 --ensemble-only > gpurun_out/r02h_c4_chi128_ensemble.log 2>&1; echo "exit $?" >> gpurun_out/r02h_c4_chi128_ensemble.log
