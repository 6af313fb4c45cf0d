# Gram loop: 2 vs 4 k-steps in flight (diagnostics builds, phase counters)
for rep in 1 2; do
  timeout 600 python tools/time_prefix.py 32 64 4 5 200 2.0 148 60 > gpurun_out/r02w_prefix60_unroll2_$rep.log 2>&1
  TB_LIB=$PWD/paper_2604_13144_b200/libtepai_b200_prof_u4.so timeout 600 python tools/time_prefix.py 32 64 4 5 200 2.0 148 60 > gpurun_out/r02w_prefix60_unroll4_$rep.log 2>&1
done
