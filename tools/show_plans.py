import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import ctypes
from paper_2512_02371_b200 import axis, filters, _lib
l = _lib.load(); o = (ctypes.c_int * 8)()
def show(name, ra, ca, planes, dt=1):
    st = l.ts_separable_plan(ra.handle, ca.handle, planes, dt, o)
    print(name, st, "nst nmid resident smem R1 nb2 tiles grid =", list(o), "K", ra.info["window"], ca.info["window"])
show("c2", axis.lanczos3(2160, 1080, 0), axis.lanczos3(3840, 1920, 0), 48)
show("c1 f32", axis.lanczos3(1080, 540, 0), axis.lanczos3(1920, 960, 0), 48, 2)
for t in (9, 15, 21, 31):
    k = filters.gaussian_taps(t)
    show(f"gauss{t}", axis.convolution(4320, k, 0), axis.convolution(7680, k, 0), 48)
show("up2x", axis.lanczos3(1080, 2160, 0), axis.lanczos3(1920, 3840, 0), 24)
from paper_2512_02371_b200 import axis as _ax
from oracle import pipelines_ref as _pr
ra = _ax.resample_filter(2160, 1080, filters.gaussian_taps(9), 0)
ca = _ax.resample_filter(3840, 1920, filters.gaussian_taps(9), 0)
show("c5 composed", ra, ca, 48)
