# round 2, session 3: TMA/LDG gather rates with a true DRAM footprint (2 GB, all column blocks), random
# and decode-shrink order; plus locate the producer-warps=6 crash
set -u
O=gpurun_out/s3rate
mkdir -p $O
PAT=0 timeout 300 .variants/tma_rate > $O/rate_pat0.txt 2>&1
PAT=1 timeout 300 .variants/tma_rate > $O/rate_pat1.txt 2>&1
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/base.so
cp .variants/libcts_pw6.so $L
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 > $O/pw6_pytest.txt 2>&1
cp /tmp/base.so $L
