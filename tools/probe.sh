#!/bin/bash
# System probe on the GPU box.
nvidia-smi; nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; ls /root/reference 2>&1 | head -2
python -c "import numba, scipy; print('numba', numba.__version__, 'scipy', scipy.__version__)"
./tools/probe_fma
