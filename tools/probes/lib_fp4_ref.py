"""Library comparison point for the MXFP4 linear: cuBLASLt (torch._scaled_mm) and
flashinfer mm_fp4 on the same M=K=N=4096 shape as BASELINE config 2, timed with
CUDA events (L2 flushed between launches).  Diagnostic only -- not the product."""

import json
import sys

import torch


def timeit(fn, iters=20, flush=None):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.add_(1)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3


def main(M=4096, K=4096, N=4096):
    dev = "cuda"
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    flops = 2.0 * M * N * K
    out = {"M": M, "K": K, "N": N}
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev)
    # cuBLASLt MXFP4 via torch._scaled_mm (scales in the 128x4 blocked layout)
    try:
        fa = a.view(torch.float4_e2m1fn_x2)
        fb = b.view(torch.float4_e2m1fn_x2)
        sa = torch.full((M * K // 32,), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        sb = torch.full((N * K // 32,), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        f = lambda: torch._scaled_mm(fa, fb.t(), sa, sb, out_dtype=torch.bfloat16)
        t = timeit(f, flush=flush)
        out["cublaslt_mxfp4_us"] = t * 1e6
        out["cublaslt_mxfp4_tflops"] = flops / t / 1e12
    except Exception as ex:  # noqa: BLE001
        out["cublaslt_mxfp4_error"] = repr(ex)[:300]
    try:
        fa = a.view(torch.float4_e2m1fn_x2)
        fb = b.view(torch.float4_e2m1fn_x2)
        sa = torch.full((M * K // 16,), 56, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        sb = torch.full((N * K // 16,), 56, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        f = lambda: torch._scaled_mm(fa, fb.t(), sa, sb, out_dtype=torch.bfloat16)
        t = timeit(f, flush=flush)
        out["cublaslt_nvfp4_us"] = t * 1e6
        out["cublaslt_nvfp4_tflops"] = flops / t / 1e12
    except Exception as ex:  # noqa: BLE001
        out["cublaslt_nvfp4_error"] = repr(ex)[:300]
    # bf16 cuBLAS for scale
    try:
        x = torch.randn(M, K, dtype=torch.bfloat16, device=dev)
        w = torch.randn(N, K, dtype=torch.bfloat16, device=dev)
        t = timeit(lambda: x @ w.t(), flush=flush)
        out["cublas_bf16_tflops"] = flops / t / 1e12
    except Exception as ex:  # noqa: BLE001
        out["cublas_bf16_error"] = repr(ex)[:300]
    if "--flashinfer" in sys.argv:
        try:
            import flashinfer

            x = torch.randn(M, K, dtype=torch.bfloat16, device=dev)
            w = torch.randn(N, K, dtype=torch.bfloat16, device=dev)
            xq, xs = flashinfer.mxfp4_quantize(x)
            wq, ws = flashinfer.mxfp4_quantize(w)
            for be in ("cudnn", "cutlass", "cute-dsl"):
                try:
                    f = lambda: flashinfer.mm_fp4(xq, wq.T, xs, ws.T, None, torch.bfloat16, None, block_size=32,
                                                  use_nvfp4=False, backend=be)
                    t = timeit(f, flush=flush)
                    out[f"flashinfer_{be}_mxfp4_tflops"] = flops / t / 1e12
                except Exception as ex:  # noqa: BLE001
                    out[f"flashinfer_{be}_error"] = repr(ex)[:300]
        except Exception as ex:  # noqa: BLE001
            out["flashinfer_error"] = repr(ex)[:300]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
    main(8192, 8192, 8192)
