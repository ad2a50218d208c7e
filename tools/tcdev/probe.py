import ctypes as C, os
import numpy as np, torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtctest.so"))
rng = np.random.default_rng(0)
def run(A, B, a_mn, b_mn, swap):
    K, N = B.shape
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros(128, N, device="cuda")
    rc = L.tc_test(C.c_void_p(dA.data_ptr()), C.c_void_p(dB.data_ptr()), C.c_void_p(dC.data_ptr()), K, N, a_mn, b_mn, swap)
    return rc, dC.cpu().numpy()
for swap in (0, 1):
    for K, N, a_mn, b_mn in [(64, 128, 1, 0), (64, 128, 0, 1), (16, 32, 1, 1)]:
        A = rng.standard_normal((128, K)).astype(np.float32); B = rng.standard_normal((K, N)).astype(np.float32)
        rc, Cc = run(A, B, a_mn, b_mn, swap)
        ref = A.astype(np.float64) @ B
        print("swap", swap, K, N, a_mn, b_mn, rc, np.abs(Cc - ref).max() / np.abs(ref).max(), np.abs(Cc).max(), flush=True)
# mapping probe for MN-major A: one-hot A, B = [I_8 | 0]
K, N = 8, 16
B = np.zeros((K, N), np.float32); B[np.arange(8), np.arange(8)] = 1
for (r, k) in [(0, 0), (1, 0), (3, 0), (4, 0), (0, 1), (0, 3), (0, 4), (5, 6), (9, 2), (33, 7)]:
    A = np.zeros((128, K), np.float32); A[r, k] = 1
    rc, Cc = run(A, B, 1, 0, 0)
    nz = np.argwhere(np.abs(Cc) > 0.5)
    print("A[%d,%d] ->" % (r, k), nz.tolist()[:4], rc, flush=True)
