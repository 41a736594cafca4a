#!/bin/bash
# r02u: P2P (CUDA IPC peer-memory) halo transport across processes on one GPU; virial test
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distmd.py -m gpu -q -x -p no:cacheprovider -k p2p > gpurun_out/pytest_p2p_r02u.txt 2>&1; tail -15 gpurun_out/pytest_p2p_r02u.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k virial > gpurun_out/pytest_vir_r02u.txt 2>&1; tail -3 gpurun_out/pytest_vir_r02u.txt
