set -u
O=gpurun_out; mkdir -p $O
timeout 300 python profiles/micro_dw.py > $O/micro_dw.log 2>&1
RNN_GEMM_SMEM_KB=225 timeout 300 python profiles/micro_dw.py > $O/micro_dw_225.log 2>&1
RNN_GEMM_SMEM_KB=100 timeout 300 python profiles/micro_dw.py > $O/micro_dw_100.log 2>&1
