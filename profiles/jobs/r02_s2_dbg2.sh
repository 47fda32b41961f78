set -u
O=gpurun_out/s2e
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
for v in "base:" "noown:-DCTS_LOCAL_NO_OWN=1" "off:-DCTS_LOCAL_T=0"; do
  tag=${v%%:*}; fl=${v#*:}
  $NV $fl -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python profiles/microbench/debug_localt.py > $O/debug_$tag.txt 2>&1
  echo "== $tag"; grep -v "^ \|Traceback\|File\|^$" $O/debug_$tag.txt | head -12
done
