# round-2 baseline on this pool: GPU suite, decode bench, per-CTA timeline of the round-1 kernel,
# and a first compute-sanitizer pass over the tiny / cfg2 shapes (fused + split paths)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/base_decode.json 2> gpurun_out/base.err
timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/base_multi.json 2>> gpurun_out/base.err
timeout 300 python bench.py --config q_proj --no-cpu-baseline > gpurun_out/base_q_proj.json 2>> gpurun_out/base.err
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name-exclude kns=relayout python profiles/microbench/sanitize_apply.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.txt
done
cp paper_2407_00066_b200/libcts.so /tmp/libcts_keep.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -DCTS_TRACE \
  -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_base.txt 2>&1
QONLY=1 N=64 C=1 R=64 T=256 timeout 300 python profiles/microbench/trace_fused.py > gpurun_out/trace_base_q.txt 2>&1
cp /tmp/libcts_keep.so paper_2407_00066_b200/libcts.so
