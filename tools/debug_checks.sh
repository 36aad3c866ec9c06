#!/bin/bash
# Bounds-checked run of the GPU test suite (compute-sanitizer is closed on the GPU
# pool): build libesnmf.so with -DESNMF_DEBUG_CHECKS=1 (every ESNMF_CHECK prints the
# failing condition and traps), put it in place of the product library, run the
# GPU tests.  Run under gpurun from the repo root; logs in gpurun_out/.
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
     -DESNMF_DEBUG_CHECKS=1 paper_1510_05237_b200/csrc/esnmf.cu -o /tmp/libesnmf_dbg.so \
     > gpurun_out/dbg_build.log 2>&1 || { echo "debug build failed"; exit 1; }
cp paper_1510_05237_b200/libesnmf.so /tmp/libesnmf_prod.so
cp /tmp/libesnmf_dbg.so paper_1510_05237_b200/libesnmf.so   # newer than the sources: no rebuild
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/dbg_tests.log 2>&1
rc=$?
cp /tmp/libesnmf_prod.so paper_1510_05237_b200/libesnmf.so
echo "debug-checked GPU tests rc=$rc" | tee -a gpurun_out/dbg_tests.log
tail -3 gpurun_out/dbg_tests.log
exit $rc
