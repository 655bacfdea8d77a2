#!/bin/bash
# CLI wall time on a 512 MiB config-1 file in /dev/shm (fix to a new file, fix in place, check).
D=/dev/shm
python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2601_06349_b200 import _lib
_lib.gen_config(1, 1 << 28, seed=1).cpu().numpy().tofile("/dev/shm/c1.bin")
PY
for i in 1 2; do
  for cmd in "fix $D/c1.bin -o $D/out.bin -e le" "fix $D/c1.bin -i -e le" "check $D/c1.bin -e le"; do
    s=$(date +%s.%N); ./paper_2601_06349_b200/u16m $cmd > /dev/null 2>&1; rc=$?; e=$(date +%s.%N)
    echo "u16m $cmd: rc=$rc $(python -c "print(round($e-$s,3))") s"
  done
done
rm -f $D/c1.bin $D/out.bin
printf 'A\0B\0' > $D/tiny.bin
for i in 1 2; do s=$(date +%s.%N); ./paper_2601_06349_b200/u16m check $D/tiny.bin -e le > /dev/null; e=$(date +%s.%N); echo "u16m check tiny: $(python -c "print(round($e-$s,3))") s"; done
python - <<'PY'
import time, ctypes
t=time.perf_counter(); L=ctypes.CDLL("./paper_2601_06349_b200/libu16m.so"); t1=time.perf_counter()
import numpy as np
x=np.zeros(4,np.uint16); o=np.zeros(4,np.uint16)
t2=time.perf_counter(); L.u16m_to_well_formed_host(ctypes.c_void_p(x.ctypes.data), ctypes.c_size_t(4), ctypes.c_void_p(o.ctypes.data)); t3=time.perf_counter()
L.u16m_to_well_formed_host(ctypes.c_void_p(x.ctypes.data), ctypes.c_size_t(4), ctypes.c_void_p(o.ctypes.data)); t4=time.perf_counter()
print(f"dlopen {t1-t:.3f}s first call (CUDA init + pipeline setup) {t3-t2:.3f}s second call {1e3*(t4-t3):.2f} ms")
PY
