# A/B of two engine builds on the same workloads (TB_LIB selects the library)
TAG=$1; shift
for lib in "$@"; do
  for rep in 1 2; do
    echo "== $lib rep $rep" >> gpurun_out/${TAG}_ab.log
    TB_LIB=$PWD/paper_2604_13144_b200/$lib TB_PROFILE=1 python tools/time_prefix.py 32 64 4 5 200 2.0 148 30 >> gpurun_out/${TAG}_ab.log 2>&1
  done
  TB_LIB=$PWD/paper_2604_13144_b200/$lib TB_PROFILE=1 python tools/prof_svd.py 148 3 >> gpurun_out/${TAG}_ab.log 2>&1
  TB_LIB=$PWD/paper_2604_13144_b200/$lib TB_PROFILE=1 python tools/time_prefix.py 16 32 2 3 200 2.0 296 60 >> gpurun_out/${TAG}_ab.log 2>&1
done
