# first run of the exchange-free decode kernel: targeted GPU tests, then the decode bench both ways
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "exchange_free or two_streams or mistral_layer or residual or deterministic or uncompressed or diagonal" > gpurun_out/t_local.txt 2>&1
tail -30 gpurun_out/t_local.txt
timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/loc_decode.json 2> gpurun_out/loc.err
CTS_LOCAL=0 timeout 300 python bench.py --config decode --steps 100 --no-cpu-baseline > gpurun_out/old_decode.json 2>> gpurun_out/loc.err
timeout 300 python bench.py --config multi --steps 50 --no-cpu-baseline > gpurun_out/loc_multi.json 2>> gpurun_out/loc.err
tail -5 gpurun_out/loc.err
