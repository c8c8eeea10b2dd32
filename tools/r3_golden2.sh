#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_golden.py -q -m gpu -rxX 2>&1 | grep -E "^E  +(Assertion|assert)|passed|failed|XFAIL" | head -8
timeout 900 python tools/c4_errors.py c3_full 2>&1 | tail -12
