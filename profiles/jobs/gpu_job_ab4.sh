set -u
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -5 > gpurun_out/pytest.txt
for m in 1 0 2; do
  for c in decode prefill; do
    CTS_EXPAND_STORE=$m timeout 300 python bench.py --config $c --steps 60 --no-cpu-baseline > gpurun_out/ab4_split1_${c}_s$m.json 2> gpurun_out/ab4_${c}_s$m.err
  done
done
$NV -DCTS_EPI_SPLIT=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
for c in decode prefill; do
  timeout 300 python bench.py --config $c --steps 60 --no-cpu-baseline > gpurun_out/ab4_split0_${c}.json 2> gpurun_out/ab4_split0_${c}.err
done
