"""Dev check of tc_common.cuh on a B200: python tools/tcdev/run_tc_test.py"""
import ctypes as C, os, subprocess, sys
import numpy as np
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libtctest.so")
L = C.CDLL(so)
rng = np.random.default_rng(0)
ok = True
for K, N, a_mn, b_mn in [(8, 32, 0, 0), (64, 128, 0, 0), (64, 128, 1, 0), (64, 128, 0, 1), (64, 256, 1, 1), (32, 64, 1, 0)]:
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros(128, N, device="cuda")
    rc = L.tc_test(C.c_void_p(dA.data_ptr()), C.c_void_p(dB.data_ptr()), C.c_void_p(dC.data_ptr()), K, N, a_mn, b_mn)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = np.abs(dC.cpu().numpy() - ref).max() / np.abs(ref).max()
    print("K=%d N=%d a_mn=%d b_mn=%d rc=%d relerr=%.3e" % (K, N, a_mn, b_mn, rc, err), flush=True)
    ok &= rc == 0 and err < 1e-6
print("ALL OK" if ok else "FAIL")
