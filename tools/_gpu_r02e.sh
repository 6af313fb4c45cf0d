bash tools/_gpu_ab.sh r02e libtepai_b200_base.so libtepai_b200_v2.so
python - > gpurun_out/r02e_maxsweep.log 2>&1 <<'PY'
import os, math, numpy as np, sys
sys.path.insert(0, ".")
os.environ["TB_MAX_SWEEPS"] = "2"
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import _lib
ham = tb.build_spin_ring(32, 1.0, 4)
run = tb.run_ensemble(ham, tb.PaiConfig(math.pi / 2**7, 30, 0.3), 5, range(8), "01" * 16, tb.TruncationPolicy(64, 1e-12), [10, 20, 30])
print("maxsweep=2 excluded:", run.excluded, "status", _lib.take_status(_lib.context(0)))
PY
python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py tests/test_postprocess.py -m gpu -q -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02e_pytest.log
