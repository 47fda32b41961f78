set -u
O=gpurun_out/s2f
mkdir -p $O
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
for v in "off:-DCTS_LOCAL_T=0" "base:"; do
  tag=${v%%:*}; fl=${v#*:}
  $NV $fl -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
  for c in one tiny qkv attn; do
    CUDA_LAUNCH_BLOCKING=1 timeout 120 python profiles/microbench/debug_localt.py $c > $O/debug_${tag}_$c.txt 2>&1
    echo "== $tag $c"; grep -v "^ \|Traceback\|File\|^$" $O/debug_${tag}_$c.txt | head -4
  done
done
timeout 300 compute-sanitizer --tool memcheck python profiles/microbench/debug_localt.py one > $O/memcheck_one.txt 2>&1
grep -m2 -B2 -A14 "Error" $O/memcheck_one.txt | head -40
