import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib
L = _lib.raw()
n = 1 << 25
x = _lib.gen_config(4, n, seed=4, shard_len=n)
w = torch.empty_like(x)
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run(name, fn):
    ts = []
    for i in range(23):
        w.copy_(x); _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); assert fn() == 0; b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[3:]); print(f"{name}: median {ts[len(ts)//2]*1e3:.1f} us", flush=True)
run("in place, plain", lambda: L.u16m_to_well_formed_in_place(w.data_ptr(), n, s))
run("in place, LE + count", lambda: L.u16m_fix_utf16_bytes(w.data_ptr(), n, w.data_ptr(), 0, cnt.data_ptr(), s))
run("in place, LE no count", lambda: L.u16m_fix_utf16_bytes(w.data_ptr(), n, w.data_ptr(), 0, None, s))
