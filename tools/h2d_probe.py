"""Host<->device copy rates from pinned memory: one stream vs two, H2D alone vs with D2H."""
import torch


def t(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)


n = 1 << 30  # 1 GiB
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    ms = t(lambda: d.copy_(h, non_blocking=True))
print("H2D 1 GiB one stream", round(n / ms / 1e6, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    half = n // 2
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for _ in range(2):
    ms = t(two)
print("H2D 1 GiB two streams", round(n / ms / 1e6, 1), "GB/s")


def duplex():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for _ in range(2):
    ms = t(duplex)
print("H2D + D2H 1 GiB each concurrently", round(2 * n / ms / 1e6, 1), "GB/s total")
