# CVAE fused decoder A/B across library builds: p50 of decode(1000) and kernel durations
mkdir -p gpurun_out/cvae_ab
for L in "$@"; do
  echo "== $L"
  BD_LIB_PATH=$L python -c "
import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_2212_02224_b200.cvae import CVAEDecoder
from oracle.cvae import decode_bf16
dec = CVAEDecoder.synthetic(7)
rng = np.random.default_rng(1)
obs = rng.standard_normal(55).astype(np.float32)
z = rng.standard_normal((1000, 2)).astype(np.float32)
for _ in range(5): out = dec.decode(obs, z)
t = []
for _ in range(200):
    t0 = time.perf_counter(); out = dec.decode(obs, z); t.append(time.perf_counter() - t0)
emu = decode_bf16(dec.W, dec.b, obs, z); sc = np.abs(emu).max()
print(f'decode p50 {np.median(t) * 1e6:.1f} us, vs bf16 restatement max {np.abs(out - emu).max() / sc:.2e}')
np.save('gpurun_out/cvae_ab/out_' + '$L'.replace('/', '_') + '.npy', out)
"
  BD_LIB_PATH=$L ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv -k regex:cvae_fused -s 5 -c 20 python -c "
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2212_02224_b200.cvae import CVAEDecoder
dec = CVAEDecoder.synthetic(7)
rng = np.random.default_rng(1)
obs = rng.standard_normal(55).astype(np.float32)
z = rng.standard_normal((1000, 2)).astype(np.float32)
for _ in range(30): dec.decode(obs, z)
" 2>/dev/null | grep cvae_fused | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | awk '{a[NR]=$1} END {print "kernel ns median", a[int(NR/2)+1], "min", a[1]}'
done
