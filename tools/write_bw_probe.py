"""HBM ceilings by access mix on this GPU (CUDA events, best of 6 over 4 GiB):
read-only (duchess_read_stream), write-only (duchess_write_stream, streaming
stores; torch fill_ for comparison) and a copy (read + write bytes)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_24957_b200 import _lib  # noqa: E402

lib = _lib.load()
n = 4 << 30
x = torch.empty(n, dtype=torch.uint8, device="cuda")
y = torch.empty(n, dtype=torch.uint8, device="cuda")
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def t(fn, reps=6):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


print("read-only  duchess_read_stream GB/s", round(n / t(lambda: lib.duchess_read_stream(
    x.data_ptr(), n, sink.data_ptr(), st)) / 1e6, 1))
print("write-only duchess_write_stream GB/s", round(n / t(lambda: lib.duchess_write_stream(
    x.data_ptr(), n, 7, st)) / 1e6, 1))
print("write-only torch fill_ GB/s", round(n / t(lambda: x.fill_(7)) / 1e6, 1))
print("copy (read + write bytes) GB/s", round(2 * n / t(lambda: y.copy_(x)) / 1e6, 1))
