# round 2, session 3: per-item expand timeline (epilogue acc ready / TMEM read / stores; MMA acc free / operands)
set -u
O=gpurun_out/s3trace
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
cp $L /tmp/final.so
cp .variants/libcts_trace.so $L
timeout 300 python profiles/microbench/trace_fused.py > $O/trace_items_detail.txt 2>&1
C=128 N=8192 timeout 300 python profiles/microbench/trace_fused.py > $O/trace_items_detail_cfg5.txt 2>&1
cp /tmp/final.so $L
cat $O/trace_items_detail.txt
