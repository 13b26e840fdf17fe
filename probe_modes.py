import json, torch
from paper_2512_02371_b200 import _lib
L = _lib.load()
g = torch.Generator(device="cpu").manual_seed(0)
res = []
cases = [(0,0,16,16),(0,0,48,16),(0,0,48,32),(0,0,64,64),(0,0,128,128),(0,0,256,256),
         (1,0,48,16),(1,1,64,128),(1,1,256,128),(1,1,256,256),(0,1,64,128),
         (2,0,48,16),(2,0,128,16),(2,0,128,64),(2,0,256,128)]
for am, bm, k, n in cases:
    a = torch.randn(128, k, generator=g).bfloat16().float().cuda()
    b = torch.randn(k, n, generator=g).bfloat16().float().cuda()
    if am == 2:  # tf32 operands: round to tf32-ish to compare
        a = torch.randn(128, k, generator=g).cuda(); b = torch.randn(k, n, generator=g).cuda()
    d = torch.zeros(128, n, device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(L.ts_probe_mma(am, bm, a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n, 1, cyc.data_ptr(), None))
    torch.cuda.synchronize()
    ref = a.double() @ b.double()
    err = ((d.double() - ref).abs().max() / ref.abs().max()).item()
    reps = 64
    _lib.check(L.ts_probe_mma(am, bm, a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n, reps, cyc.data_ptr(), None))
    torch.cuda.synchronize()
    kstep = 8 if am == 2 else 16
    nm = reps * k // kstep
    res.append({"amode": am, "bmode": bm, "k": k, "n": n, "rel_err": err, "cyc_per_mma": cyc.item() / nm,
                "macs_per_cyc": 128 * n * kstep / (cyc.item() / nm)})
    print(json.dumps(res[-1]))
