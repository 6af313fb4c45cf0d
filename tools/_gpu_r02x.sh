# final build: whole GPU suite, smoke, bench (both arms)
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02x_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02x_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02x_smoke.log 2>&1
python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; echo "bench exit $?" >> gpurun_out/r02x_bench.err
python bench.py --impl reference > gpurun_out/r02x_bench_reference_arm.json 2> gpurun_out/r02x_bench_reference_arm.err
