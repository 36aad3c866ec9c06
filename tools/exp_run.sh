# development: GPU suite + alternating timings (quick_time) under gpurun
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests3.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests3.log
for i in 1 2 3; do
python tools/quick_time.py --steps 50 --warmup 6 --tag new >> gpurun_out/exp4.log 2>&1
ESNMF_NO_POLISH_SPLIT=1 python tools/quick_time.py --steps 50 --warmup 6 --tag nosplit >> gpurun_out/exp4.log 2>&1
ESNMF_NO_POLISH_SPLIT=1 ESNMF_VPREP_MAIN=1 python tools/quick_time.py --steps 50 --warmup 6 --tag old >> gpurun_out/exp4.log 2>&1
done
