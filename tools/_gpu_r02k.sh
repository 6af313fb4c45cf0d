# debug of the cluster-Jacobi orthogonality at 129x129 (graded, preconditioned)
timeout 600 python tools/dbg_cluster129.py > gpurun_out/r02k_dbg_cluster.log 2>&1; echo "exit $?" >> gpurun_out/r02k_dbg_cluster.log
