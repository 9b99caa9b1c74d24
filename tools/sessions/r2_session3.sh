#!/bin/bash
# round-2 GPU session 3 (2 GPUs): spectral parity vs reference goldens, full-size parity vs the reference
O=gpurun_out/s3
mkdir -p $O
df -h /tmp . /dev/shm > $O/df.txt 2>&1
timeout 600 python -m pytest tests/test_spectral_golden.py -m gpu -q -s > $O/pytest_spectral.log 2>&1; echo "exit $?" >> $O/pytest_spectral.log
timeout 1200 python -m pytest tests/test_fullsize_ref.py -m gpu -q -s > $O/pytest_fullsize.log 2>&1; echo "exit $?" >> $O/pytest_fullsize.log
echo done
