import torch, json
from paper_2512_02371_b200 import _lib
L = _lib.load()
g = torch.Generator(device="cpu").manual_seed(0)
for am, k, n in [(2, 16, 16), (3, 16, 16), (3, 32, 16), (3, 128, 16), (4, 16, 16), (4, 128, 16)]:
    a = torch.randn(128, k, generator=g).cuda(); b = torch.randn(k, n, generator=g).cuda()
    d = torch.zeros(128, n, device="cuda")
    _lib.check(L.ts_probe_mma(am, 0, a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n, 1, None, 1, None))
    torch.cuda.synchronize()
    ref = a.double() @ b.double()
    print(json.dumps({"amode": am, "k": k, "n": n, "rel_err": ((d.double() - ref).abs().max() / ref.abs().max()).item(), "dmax": d.abs().max().item()}))
