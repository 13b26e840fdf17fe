import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2512_02371_b200 import pipelines, _lib
L = _lib.load()
rng = np.random.default_rng(0)
x = rng.random((1, 128, 128), dtype=np.float32)
xt = torch.from_numpy(x).bfloat16().cuda()
dbg = torch.zeros(4 * 2 * 128 * 256, device="cuda")
_lib.check(L.ts_debug_dct16(dbg.data_ptr()))
y = pipelines.denoise_dct16(xt, threshold=0.0, mode="soft", out_dtype=torch.float32)
torch.cuda.synchronize()
_lib.check(L.ts_debug_dct16(None))
np.savez("gpurun_out/dbg_dct.npz", x=xt.float().cpu().numpy(), y=y.cpu().numpy(), dbg=dbg.view(4, 2, 128, 256).cpu().numpy())
print("ok", float(y.abs().max()))
