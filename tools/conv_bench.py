"""Back-to-back launch timing of one conv shape through the kernel hook vs the
same shape inside an executor layer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
from paper_2304_09961_b200._native import bs_conv_desc, check, exec_lib, fptr

def bench(nimg, H, Cin, N, k, pad, in_ldc=None, reps=50, split=1, res=False, stride=1):
    in_ldc = in_ldc or Cin
    Ho = (H + 2 * pad - k) // stride + 1
    x = np.random.default_rng(0).standard_normal((nimg, H, H, in_ldc)).astype(np.float32)
    K = k * k * Cin; Kp = (K + 31) // 32 * 32
    w = np.zeros((N, Kp), np.float32); b = np.zeros(N, np.float32)
    out = np.zeros((nimg, Ho, Ho, N), np.float32)
    r = np.random.default_rng(1).standard_normal((nimg, Ho, Ho, N)).astype(np.float32) if res else None
    d = bs_conv_desc(H=H, W=H, Cin=Cin, Ho=Ho, Wo=Ho, KH=k, KW=k, stride=stride, pad=pad, N=N, in_ldc=in_ldc, in_coff=0,
                     out_ldc=N, out_coff=0, res_ldc=N, res_coff=0, relu=1, round_out=0, split=split)
    ms = C.c_float()
    check(exec_lib().bs_kernel_conv(d, nimg, fptr(x), fptr(w), fptr(b), fptr(r) if res else None, fptr(out), reps, C.byref(ms)))
    return ms.value * 1000

if __name__ == "__main__":
    for split in (1, 0):
        for nimg in (1, 8, 90):
            print(f"split={split} b={nimg:2d} 3x3 14x14 128->256: {bench(nimg, 14, 128, 256, 3, 1, split=split):7.1f} us   "
                  f"1x1 7x7 832->384: {bench(nimg, 7, 832, 384, 1, 0, split=split):7.1f} us", flush=True)
    from paper_2304_09961_b200.executor import Executor
    with Executor("googlenet", max_batch=90, max_requests=4) as ex:
        for nimg in (1, 8, 90):
            print(f"executor layer 13 (i4c_b) b={nimg}: {ex.profile_layer(0, 13, nimg, 20) * 1000:7.1f} us", flush=True)
