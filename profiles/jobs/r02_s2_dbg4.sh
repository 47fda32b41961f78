set -u
O=gpurun_out/s2g
mkdir -p $O
for c in 527930e ebc37ea; do
  CTS_PKG_ROOT=dbg_so/pkg_$c CUDA_LAUNCH_BLOCKING=1 timeout 120 python profiles/microbench/debug_localt.py one tiny > $O/debug_$c.txt 2>&1
  echo "== $c"; grep -v "^ \|Traceback\|File\|^$" $O/debug_$c.txt | head -4
done
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
$NV -DCTS_DEBUG_OWN_POLL=1 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
CTS_EARLY_ITEMS=0 CUDA_LAUNCH_BLOCKING=1 timeout 120 python profiles/microbench/debug_localt.py tiny > $O/debug_ownpoll.txt 2>&1
echo "== ownpoll"; grep -v "^ \|Traceback\|File\|^$" $O/debug_ownpoll.txt | head -4
