set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k "projection" -x -q > $O/pytest_proj.log 2>&1; echo "exit $?" >> $O/pytest_proj.log
timeout 300 python profiles/probe_gemm.py > $O/probe_gemm.log 2>&1
timeout 300 python profiles/micro_dw.py > $O/micro_dw.log 2>&1
RNN_NO_DWT=1 timeout 300 python profiles/micro_dw.py > $O/micro_dw_nodwt.log 2>&1
RNN_GEMM_SMEM_KB=100 timeout 300 python profiles/micro_dw.py > $O/micro_dw_100.log 2>&1
bash profiles/run_dhnvar.sh
