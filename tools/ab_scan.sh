cd "$(dirname "$0")/.."
./tools/gpu_check.sh | grep -E "TESTS|BENCH|FAIL"
GIVF_SCAN=legacy ./tools/gpu_check.sh | grep -E "BENCH"
