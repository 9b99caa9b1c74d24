#!/bin/bash
# round-2 GPU session 71 (2 GPUs): final-code config D (1024^3 C2C fp64 pencil 4x2, 8 ranks over 2 B200s) vs the unmodified reference
O=gpurun_out/s71
mkdir -p $O
timeout 1500 env DFFTB_TEST_HUGE=1 python -m pytest tests/test_fullsize_ref.py -m gpu -q -s -k huge > $O/pytest_huge.log 2>&1; echo "exit $?" >> $O/pytest_huge.log
grep -E "case|passed|failed|exit" $O/pytest_huge.log
echo done
