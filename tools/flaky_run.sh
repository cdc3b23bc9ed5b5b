for i in 1 2 3 4; do timeout 600 python -m pytest -q tests -m gpu --tb=short 2>&1 | grep -E "^E  |^FAILED|passed|failed|assert rel_err|AssertionError" | head -8; done
