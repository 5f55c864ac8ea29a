"""Is PCIe full duplex here?  1.2 GB H2D alone, 268 MB D2H alone, and both
at once on two streams (pinned host buffers)."""
import torch

h_up = torch.empty(1_200_000_000, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty_like(h_up, device="cuda")
d_dn = torch.empty(268_435_456, dtype=torch.uint8, device="cuda")
h_dn = torch.empty(268_435_456, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def up():
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def dn():
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


print(f"H2D 1.2 GB alone {t(up):.2f} ms, D2H 268 MB alone {t(dn):.2f} ms, both {t(both):.2f} ms")
