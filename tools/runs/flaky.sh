for v in "NPSD_COARSE_ZC=8" "NPSD_COARSE_OLD=1" "NPSD_COARSE_ZC=8" "NPSD_COARSE_OLD=1"; do
echo "== $v"; env $v timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|^E  |FAILED" | head -5
done
