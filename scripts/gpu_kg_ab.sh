mkdir -p gpurun_out
rm -f gpurun_out/variants.log
for r in 1 2; do
MODE=pick bash scripts/gpu_variants.sh "" $PWD/build_variants/liborloj_kg1.so $PWD/build_variants/liborloj_kg2.so $PWD/build_variants/liborloj_kg4.so
done
ORLOJ_LIB=$PWD/build_variants/liborloj_kg1.so timeout 600 python -m pytest -q -x tests/test_gpu_score.py tests/test_gpu_invariants.py > gpurun_out/pytest_kg1.log 2>&1; echo rc=$? >> gpurun_out/pytest_kg1.log
