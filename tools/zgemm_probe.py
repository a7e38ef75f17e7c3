"""FP64 complex GEMM rates for C5's rank-32 LowRank halves on this box:
torch (cuBLAS ZGEMM) and cublasZgemm3m (Gauss 3-multiply) through ctypes, vs
the shapes W = V^H X (32 x 1e6 x 128) and Y += U W (1e6 x 32 x 128)."""
import ctypes
import torch

N, K, r = 1000003, 128, 32
dev = "cuda"
X = torch.randn(N, K, dtype=torch.complex128, device=dev)
V = torch.randn(N, r, dtype=torch.complex128, device=dev)
U = torch.randn(N, r, dtype=torch.complex128, device=dev)
Y = torch.randn(N, K, dtype=torch.complex128, device=dev)
W = torch.empty(r, K, dtype=torch.complex128, device=dev)


def t(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("torch contract V^H X:", t(lambda: torch.mm(V.mH, X)), "ms")
Wt = torch.mm(V.mH, X)
print("torch expand Y += U W:", t(lambda: Y.addmm_(U, Wt)), "ms")

import nvidia.cublas, os  # noqa: E401
lib = ctypes.CDLL(os.path.join(os.path.dirname(nvidia.cublas.__file__), "lib", "libcublas.so.12"))
h = ctypes.c_void_p()
assert lib.cublasCreate_v2(ctypes.byref(h)) == 0
lib.cublasSetStream_v2(h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
one = (ctypes.c_double * 2)(1.0, 0.0)
zero = (ctypes.c_double * 2)(0.0, 0.0)
OP_N, OP_C = 0, 2
for name in ("cublasZgemm_v2", "cublasZgemm3m"):
    fn = getattr(lib, name)
    # W' (K x r, ld K) = X' (K x N, ld K) * V'^H  (V' = r x N, ld r)
    def contract():
        st = fn(h, OP_N, OP_C, K, r, N, one, ctypes.c_void_p(X.data_ptr()), K, ctypes.c_void_p(V.data_ptr()), r,
                zero, ctypes.c_void_p(W.data_ptr()), K)
        assert st == 0, st
    # Y' (K x N) += W' (K x r) * U' (r x N)
    def expand():
        st = fn(h, OP_N, OP_N, K, N, r, one, ctypes.c_void_p(W.data_ptr()), K, ctypes.c_void_p(U.data_ptr()), r,
                one, ctypes.c_void_p(Y.data_ptr()), K)
        assert st == 0, st
    print(name, "contract:", t(contract), "ms  expand(+=):", t(expand), "ms")
    contract()
    torch.cuda.synchronize()
    print("   contract rel err vs torch:", float((W - Wt).abs().max() / Wt.abs().max()))
