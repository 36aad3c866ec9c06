# development: timings (quick_time) under gpurun, then the GPU suite
mkdir -p gpurun_out
for i in 1 2 3; do
python tools/quick_time.py --steps 50 --warmup 6 --tag pair2 >> gpurun_out/exp9.log 2>&1
done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests9.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests9.log
