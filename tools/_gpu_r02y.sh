# final build: ncu counters + launch list of the bench step; whole-config C1 / C2 / C4 chi=16 runs
bash tools/ncu_ensemble_metrics.sh r02y > gpurun_out/r02y_ncu_script.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/r02y_launches_bench_steps1_warmup3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02y_ncu_launchlist.log 2>&1
timeout 300 python tools/run_config.py C1 > gpurun_out/r02y_config_c1.log 2>&1
timeout 900 python tools/run_config.py C2 > gpurun_out/r02y_config_c2.log 2>&1
timeout 600 python tools/time_c4.py 16 592 750 > gpurun_out/r02y_c4_chi16_full.log 2>&1
