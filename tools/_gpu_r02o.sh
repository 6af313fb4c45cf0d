timeout 600 python tools/dbg_small_c4.py 592 100 0 1 > gpurun_out/r02o_plain.log 2>&1; echo "exit $?" >> gpurun_out/r02o_plain.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/dbg_small_c4.py 8 30 1 > gpurun_out/r02o_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/r02o_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/dbg_small_c4.py 4 12 1 > gpurun_out/r02o_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/r02o_racecheck.log
