#!/bin/bash
# Negative control for the slow-reader SPMD test: rebuild a copy WITHOUT the remote-reader
# WAR bookkeeping and check that the test then fails.
set -u
rm -rf /tmp/neg && cp -r . /tmp/neg && cd /tmp/neg
sed -i '/for (const PendEntry& e : ep->reads) ctx->pend/d' paper_1809_05657_b200/csrc/hda.cpp
python -m paper_1809_05657_b200.build > /dev/null 2>&1 || { echo "neg build failed"; exit 1; }
timeout 600 python -m pytest tests/test_gpu_spmd.py -q -k "slow" 2>&1 | tail -3
