set -x
nvidia-smi -L
python -c "import torch; print(torch.cuda.is_available())"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/t1.log
cat gpurun_out/t1.log | tail -40
