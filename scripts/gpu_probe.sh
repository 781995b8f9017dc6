mkdir -p gpurun_out
(nproc; free -g; lscpu | head -30; nvidia-smi; df -h /tmp /dev/shm) > gpurun_out/box_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02_start.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02_start.log
