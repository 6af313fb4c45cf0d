bash tools/_gpu_ab.sh r02f libtepai_b200_v2.so libtepai_b200_v4.so
python - > gpurun_out/r02f_maxsweep.log 2>&1 <<'PY'
import os, math, numpy as np, sys
sys.path.insert(0, ".")
os.environ["TB_MAX_SWEEPS"] = "2"
import paper_2604_13144_b200 as tb
ham = tb.build_spin_ring(32, 1.0, 4)
run = tb.run_ensemble(ham, tb.PaiConfig(math.pi / 2**7, 30, 0.3), 5, range(8), "01" * 16, tb.TruncationPolicy(64, 1e-12), [10, 20, 30])
print("maxsweep=2 excluded:", run.excluded)
PY
python -m pytest tests -m gpu -q -p no:cacheprovider -k "not c3_stat and not truncated_statistics" > gpurun_out/r02f_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02f_pytest.log
