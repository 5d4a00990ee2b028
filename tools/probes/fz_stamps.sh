# CTA 0's phase stamps of the fused CVAE kernel (BD_PHASE_TIMING builds), warm, per library
for L in "$@"; do
  echo "== $L"
  BD_LIB_PATH=$L python -c "
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2212_02224_b200.cvae import CVAEDecoder
dec = CVAEDecoder.synthetic(7)
rng = np.random.default_rng(1)
obs = rng.standard_normal(55).astype(np.float32)
z = rng.standard_normal((1000, 2)).astype(np.float32)
for _ in range(6): dec.decode(obs, z)
" 2>&1 | grep FZ | tail -2
done
