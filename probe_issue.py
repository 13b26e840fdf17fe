import torch, json
from paper_2512_02371_b200 import _lib
L = _lib.load()
names = ["N16 acc1", "N16 acc8", "N64 acc1", "N64 acc4", "N256 acc1", "N256 acc2"]
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for v in range(6):
    for rep in range(3):
        _lib.check(L.ts_probe_issue(v, c.data_ptr(), None)); torch.cuda.synchronize()
    print(json.dumps({"variant": names[v], "cycles_64_mma": c.item(), "cyc_per_mma": c.item() / 64}))
names = ["TS N16 f16", "TS N64 f16", "TS N16 tf32", "TS N64 tf32"]
for v in range(4):
    for rep in range(3):
        _lib.check(L.ts_probe_issue_ts(v, c.data_ptr(), None)); torch.cuda.synchronize()
    print(json.dumps({"variant": names[v], "cycles_64_mma": c.item(), "cyc_per_mma": c.item() / 64}))
