# round 2, session 3: stacked-space JD on a rank-deficient cluster (8 copies of a rank-4 LoRA, r = 16)
set -u
O=gpurun_out/s3kdup
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "rank_deficient" --timeout 300 > $O/pytest.txt 2>&1; tail -25 $O/pytest.txt
