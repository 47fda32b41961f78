set -u
O=gpurun_out/s2h
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
for v in "off:-DCTS_LOCAL_T=0" "base:"; do
  tag=${v%%:*}; fl=${v#*:}
  $NV $fl -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python profiles/microbench/debug_localt.py one > $O/debug_${tag}.txt 2>&1
  echo "== $tag split-ref"; grep -v "^ \|Traceback\|File\|^$" $O/debug_${tag}.txt | head -3
  FUSED_ONLY=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python profiles/microbench/debug_localt.py one tiny qkv > $O/debugf_${tag}.txt 2>&1
  echo "== $tag fused-only"; grep -v "^ \|Traceback\|File\|^$" $O/debugf_${tag}.txt | head -8
done
