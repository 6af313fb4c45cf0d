# final-build evidence: ncu counters + launch list of the bench step, reference arm (with the unmodified reference), C5 t0 and C4 Trotter on the cluster path
bash tools/ncu_ensemble_metrics.sh r02s > gpurun_out/r02s_ncu_script.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02s_plain_launchlist.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/r02s_launches_bench_steps1_warmup3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02s_ncu_launchlist.log 2>&1
python bench.py --impl reference > gpurun_out/r02s_bench_reference_arm.json 2> gpurun_out/r02s_bench_reference_arm.err
timeout 1200 python tools/run_c5_full.py t0 gpurun_out/c5_t0_r02s.mps > gpurun_out/r02s_c5_t0.log 2>&1; echo "exit $?" >> gpurun_out/r02s_c5_t0.log
timeout 1500 python tools/run_c4_full.py 128 148 --trotter-only > gpurun_out/r02s_c4_trotter_chi128.log 2>&1; echo "exit $?" >> gpurun_out/r02s_c4_trotter_chi128.log
