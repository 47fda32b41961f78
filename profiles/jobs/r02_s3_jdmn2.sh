# round 2, session 3: MN-major descriptor strides (LBO / SBO) probe on the failing JD case
set -u
O=gpurun_out/s3jdmn2
mkdir -p $O
L=paper_2407_00066_b200/libcts.so
for v in a b c d; do
  cp .variants/libcts_mn$v.so $L
  timeout 300 python -m pytest "tests/test_gpu_parity.py::test_gpu_jd_eigen_iteration" -q -m gpu --timeout 120 > $O/mn_$v.txt 2>&1
  echo "$v $(tail -1 $O/mn_$v.txt) $(grep -o 'AssertionError: np.float64([0-9.e-]*)' $O/mn_$v.txt | head -3 | tr '\n' ' ')"
done
