# development: alternating timings (quick_time) under gpurun, then the GPU suite
mkdir -p gpurun_out
for i in 1 2 3; do
python tools/quick_time.py --steps 50 --warmup 6 --tag new >> gpurun_out/exp5.log 2>&1
ESNMF_VROWS=1 python tools/quick_time.py --steps 50 --warmup 6 --tag vrows >> gpurun_out/exp5.log 2>&1
done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests5.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests5.log
