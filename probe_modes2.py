import json, torch
from paper_2512_02371_b200 import _lib
L = _lib.load()
g = torch.Generator(device="cpu").manual_seed(0)
cases = []
for n in (16, 32, 64, 128, 256):
    for nacc in (1, 2, 4, 8, 16):
        if nacc * n <= 512: cases.append((0, 0, 16, n, nacc))
for n in (16, 64):
    for nacc in (1, 4, 8):
        cases.append((2, 0, 16, n, nacc))
cases += [(1, 1, 16, 128, 1), (1, 1, 16, 128, 4), (1, 1, 16, 256, 2)]
for am, bm, k, n, nacc in cases:
    a = torch.randn(128, k, generator=g).bfloat16().float().cuda()
    b = torch.randn(k, n, generator=g).bfloat16().float().cuda()
    d = torch.zeros(128, n, device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    reps = 128
    _lib.check(L.ts_probe_mma(am, bm, a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n, reps, cyc.data_ptr(), nacc, None))
    torch.cuda.synchronize()
    ref = (a.double() @ b.double()) * (reps // nacc)
    err = ((d.double() - ref).abs().max() / ref.abs().max()).item()
    kstep = 8 if am == 2 else 16
    nm = reps * k // kstep
    print(json.dumps({"amode": am, "bmode": bm, "k": k, "n": n, "nacc": nacc, "rel_err": round(err, 6),
                      "cyc_per_mma": round(cyc.item() / nm, 1), "macs_per_cyc": round(128 * n * kstep / (cyc.item() / nm), 1)}))
