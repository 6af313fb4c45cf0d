bash tools/_gpu_ab.sh r02d libtepai_b200_base.so libtepai_b200.so
python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02d_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02d_pytest.log
