#!/bin/bash
# Multi-rank driver (Team): pairs in the partitioned schedule, loopback + one-rank NCCL; full suite.
O=gpurun_out/team
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -x > $O/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $O/pytest_dist.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
