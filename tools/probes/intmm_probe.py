import torch, time
a = torch.randint(-128, 128, (2048, 4096), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 128, (4096, 4096), dtype=torch.int8, device="cuda")
c = torch._int_mm(a, b)
torch.cuda.synchronize()
ref = (a.double() @ b.double()).long()
print("exact", torch.equal(c.long(), ref))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): c = torch._int_mm(a, b)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print("int_mm ms", ms, "TOPS", 2 * 2048 * 4096 * 4096 / ms / 1e9)
