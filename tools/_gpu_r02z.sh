# ncu --set full of the batched 128x128 svd_kernel on the final build (same Jacobi / TMEM-QRCP / Gram-screen code as the ensemble kernel)
TB_LIB=$PWD/paper_2604_13144_b200/libtepai_b200.so TB_PROFILE=0 python tools/prof_svd.py 148 2 > gpurun_out/r02z_plain.log 2>&1
TB_LIB=$PWD/paper_2604_13144_b200/libtepai_b200.so TB_PROFILE=0 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:svd_kernel -s 1 -c 1 -o gpurun_out/r02z_svd python tools/prof_svd.py 148 2 > gpurun_out/r02z_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r02z_svd.ncu-rep > gpurun_out/r02z_ncu_svd_kernel_summary.txt 2>&1
