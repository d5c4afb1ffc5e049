# compute-sanitizer is closed on this pool: the library's own guards instead.
#   KOT_POISON=1  fresh device allocations filled with NaN (uninitialised reads surface as NaN / test failures)
#   KOT_POISON=2  fresh allocations filled with 0x55 bytes
#   KOT_CANARY=1  64 KB guard bands around every allocation, checked on free and before every solver iteration
for mode in "KOT_POISON=1 KOT_CANARY=1" "KOT_POISON=2 KOT_CANARY=1"; do
  echo "== $mode: tools/sanitize_case.py"
  env $mode timeout 600 python tools/sanitize_case.py 2>&1 | tail -8
  echo "== $mode: pytest -m gpu (parity suites)"
  env $mode timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_api.py -m gpu -q 2>&1 | tail -3
done
