"""H2D bandwidth on the box: one large DMA copy from pinned memory, many 256 KB
DMA copies, and the zero-copy gather kernel (duchess_gather_active).
Measured (B200 box, this round): one DMA 55.5 GB/s, 4096 x 256 KB DMAs 29.9,
256 x 4 MB DMAs 52.6, zero-copy gather 50.7-51.4; a TMA-bulk (cp.async.bulk
from the host mapping through shared memory) gather variant measured the same
51.3 GB/s, so SM-initiated PCIe reads sit at ~0.93 of one large DMA."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2509_24957_b200 import _lib  # noqa: E402

rows, row_bytes = 4096, 262144
host = torch.randint(0, 255, (rows * row_bytes,), dtype=torch.uint8).pin_memory()
dev = torch.empty(rows * row_bytes, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def bw(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return rows * row_bytes * n / (time.perf_counter() - t) / 1e9


print("one DMA copy      GB/s", bw(lambda: dev.copy_(host, non_blocking=True)))
hv = host.view(rows, row_bytes)
dv = dev.view(rows, row_bytes)
print("4096 row DMAs     GB/s", bw(lambda: [dv[i].copy_(hv[i], non_blocking=True) for i in range(rows)]))
hv2 = host.view(rows // 16, 16 * row_bytes)
dv2 = dev.view(rows // 16, 16 * row_bytes)
print("256 x 4 MB DMAs   GB/s", bw(lambda: [dv2[i].copy_(hv2[i], non_blocking=True) for i in range(rows // 16)]))
lib = _lib.load()
lst = torch.arange(rows, dtype=torch.int32, device="cuda").repeat(2)      # both list parities
cnt = torch.tensor([rows, rows, 0, 0], dtype=torch.int32, device="cuda")


def gather():
    _lib.check(lib.duchess_gather_active(host.data_ptr(), dev.data_ptr(), row_bytes, lst.data_ptr(),
                                         cnt.data_ptr(), rows, _lib.stream_handle()), "gather")


print("zero-copy gather  GB/s", bw(gather))

