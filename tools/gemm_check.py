"""Standalone GPU check of the tcgen05 grouped GEMM against torch fp32 (dev tool)."""
import ctypes, sys, time
import torch

lib = ctypes.CDLL("paper_2304_11414_b200/lib/libppmoe.so")
P, I = ctypes.c_void_p, ctypes.c_int
lib.ppmoe_gemm_selftest.argtypes = [I, I, I, P, P, P, I, I, I, I, I, P, P]
lib.ppmoe_last_error.restype = ctypes.c_char_p

def seg_from_counts(counts):
    seg = [0]
    for c in counts:
        seg.append(seg[-1] + ((c + 127) // 128) * 128)
    return seg

def run(mode, use_tc, counts, M, N, K):
    dev = "cuda"
    G = len(counts)
    seg = seg_from_counts(counts)
    rows = seg[-1]
    segt = torch.tensor(seg, dtype=torch.int32, device=dev)
    torch.manual_seed(0)
    st = torch.cuda.current_stream().cuda_stream
    if mode == 0:
        A = torch.randn(rows, K, device=dev).bfloat16()
        B = torch.randn(G * K, N, device=dev).bfloat16()
        D = torch.full((rows, N), float("nan"), device=dev)
        rc = lib.ppmoe_gemm_selftest(0, use_tc, 0, A.data_ptr(), B.data_ptr(), segt.data_ptr(), G, 0, N, K, rows, D.data_ptr(), st)
        ref = torch.cat([A[seg[g]:seg[g+1]].float() @ B[g*K:(g+1)*K].float() for g in range(G)])
    elif mode == 1:
        A = torch.randn(rows, M, device=dev).bfloat16()
        B = torch.randn(rows, N, device=dev).bfloat16()
        D = torch.full((G, M, N), float("nan"), device=dev)
        rc = lib.ppmoe_gemm_selftest(1, use_tc, 0, A.data_ptr(), B.data_ptr(), segt.data_ptr(), G, M, N, 0, rows, D.data_ptr(), st)
        ref = torch.stack([A[seg[g]:seg[g+1]].float().T @ B[seg[g]:seg[g+1]].float() for g in range(G)])
    else:
        A = torch.randn(rows, K, device=dev).bfloat16()
        B = torch.randn(G * N, K, device=dev).bfloat16()
        D = torch.full((rows, N), float("nan"), device=dev)
        rc = lib.ppmoe_gemm_selftest(2, use_tc, 0, A.data_ptr(), B.data_ptr(), segt.data_ptr(), G, 0, N, K, rows, D.data_ptr(), st)
        ref = torch.cat([A[seg[g]:seg[g+1]].float() @ B[g*N:(g+1)*N].float().T for g in range(G)])
    if rc != 0:
        print("ERR", rc, lib.ppmoe_last_error()); return False
    torch.cuda.synchronize()
    err = (D - ref).abs().max().item() / max(1.0, ref.abs().max().item())
    print(f"mode={mode} tc={use_tc} counts={counts} M={M} N={N} K={K}: rel_err={err:.3e} nan={torch.isnan(D).any().item()}")
    return err < 1e-3

ok = True
for use_tc in (0, 1):
    ok &= run(0, use_tc, [128], 0, 256, 64)
    ok &= run(0, use_tc, [100, 300, 0, 5], 0, 512, 256)
    ok &= run(2, use_tc, [128], 0, 256, 64)
    ok &= run(2, use_tc, [200, 33], 0, 512, 320)
    ok &= run(1, use_tc, [128], 128, 256, 0)
    ok &= run(1, use_tc, [250, 0, 77], 256, 512, 0)
print("ALL_OK" if ok else "FAILED")
# timing of a big mode-0 GEMM
if ok:
    G, K, N = 8, 4096, 16384
    counts = [4096] * G
    seg = seg_from_counts(counts); rows = seg[-1]
    segt = torch.tensor(seg, dtype=torch.int32, device="cuda")
    A = torch.randn(rows, K, device="cuda").bfloat16(); B = torch.randn(G*K, N, device="cuda").bfloat16()
    D = torch.empty(rows, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.ppmoe_gemm_selftest(0, 1, 0, A.data_ptr(), B.data_ptr(), segt.data_ptr(), G, 0, N, K, rows, D.data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lib.ppmoe_gemm_selftest(0, 1, 0, A.data_ptr(), B.data_ptr(), segt.data_ptr(), G, 0, N, K, rows, D.data_ptr(), st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"big GEMM {rows}x{N}x{K} x{G}: {ms:.3f} ms, {2*rows*N*K/ms/1e9:.1f} TFLOP/s")
    Ab = A[:4096]; Bb = B[:K]
    for _ in range(3): torch.matmul(Ab, Bb)
    e0.record()
    for _ in range(5*G): torch.matmul(Ab, Bb)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"torch.matmul same work: {ms:.3f} ms, {2*rows*N*K/ms/1e9:.1f} TFLOP/s")
