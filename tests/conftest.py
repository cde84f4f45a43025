"""Shared pytest configuration: registers the ``gpu`` marker.

``-m "not gpu"`` runs on the CPU-only build container (oracle vs golden
vectors, host logic, C-ABI exports, multi-rank gloo sharding);
``-m gpu`` runs the CUDA parity tests on a B200."""

import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

torch.set_num_threads(min(8, os.cpu_count() or 1))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
