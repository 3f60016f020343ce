import ctypes as C, time, torch, sys, os
sys.path.insert(0, "/root/repo")
from paper_2409_02423_b200 import _lib
torch.cuda.set_device(0)
n = 1 << 24
codec = _lib.Codec(2, 8)
w = C.c_uint64(); _lib.hccx_wire_size_bytes(codec, n, C.byref(w)); W = w.value
sets = 8
xs = [torch.randn(n, device="cuda") * 1e-3 for _ in range(sets)]
ps = [torch.empty(W, dtype=torch.uint8, device="cuda") for _ in range(sets)]
ys = [torch.empty(n, device="cuda") for _ in range(sets)]
s = torch.cuda.current_stream().cuda_stream
for i in range(10):
    _lib.hccx_compress(codec, xs[i % sets].data_ptr(), n, ps[i % sets].data_ptr(), None, s)
torch.cuda.synchronize()
# host issue rate
torch.cuda._sleep(int(50e6))
t = time.perf_counter()
for i in range(200):
    _lib.hccx_compress(codec, xs[i % sets].data_ptr(), n, ps[i % sets].data_ptr(), None, s)
host_us = (time.perf_counter() - t) / 200 * 1e6
torch.cuda.synchronize()
# device time: long sleep first, then 200 back-to-back compress
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(50e6))
a.record()
for i in range(200):
    _lib.hccx_compress(codec, xs[i % sets].data_ptr(), n, ps[i % sets].data_ptr(), None, s)
b.record()
torch.cuda.synchronize()
dev_us = a.elapsed_time(b) / 200 * 1e3
# graph
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g.capture_begin()
    for i in range(20):
        _lib.hccx_compress(codec, xs[i % sets].data_ptr(), n, ps[i % sets].data_ptr(), None, st.cuda_stream)
    g.capture_end()
torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
a.record(); 
for _ in range(10): g.replay()
b.record(); torch.cuda.synchronize()
graph_us = a.elapsed_time(b) / 200 * 1e3
# same for decompress
torch.cuda._sleep(int(50e6))
a.record()
for i in range(200):
    _lib.hccx_decompress(codec, ps[i % sets].data_ptr(), W, n, ys[i % sets].data_ptr(), s)
b.record(); torch.cuda.synchronize()
dec_us = a.elapsed_time(b) / 200 * 1e3
print(dict(host_issue_us=round(host_us,2), compress_b2b_us=round(dev_us,2), compress_graph_us=round(graph_us,2), decompress_b2b_us=round(dec_us,2)))
