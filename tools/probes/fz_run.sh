mkdir -p gpurun_out/t21
BD_LIB_PATH=build_variants/lib_phase.so python -c "
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2212_02224_b200.cvae import CVAEDecoder
dec = CVAEDecoder.synthetic(7)
rng = np.random.default_rng(1)
obs = rng.standard_normal(55).astype(np.float32)
z = rng.standard_normal((1000, 2)).astype(np.float32)
for _ in range(4): dec.decode(obs, z)
" 2>&1 | grep FZ | tail -2 > gpurun_out/t21/fz.txt
python -m pytest tests/test_gpu_cvae.py -x -q > gpurun_out/t21/tests.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:cvae_fused python tools/probes/cvae_time.py > gpurun_out/t21/ncu.csv 2>&1
