set -x
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02b_pytest_gpu.log
TB_PROFILE=1 python tools/time_prefix.py 32 64 4 5 200 2.0 148 20 > gpurun_out/r02b_prefix20.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ensemble_kernel -c 1 -o gpurun_out/r02b_prof python tools/time_prefix.py 32 64 4 5 200 2.0 148 20 > gpurun_out/r02b_ncu.log 2>&1
echo done
