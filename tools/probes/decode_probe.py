"""Decode probe (C4): per-layer time of a 16-layer CUDA graph for
 lin   : linear only on pre-quantized codes,
 two   : quantize kernel + linear kernel,
 fused : serq_forward_mx (quantizer inside the decode kernel),
for SERQ_DEC_S (CTAs per weight tile) variants."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B, _lib

layers = 16
variants = os.environ.get("VARIANTS", "auto,1,2,3,4,6,8").split(",")
SHAPES = [tuple(int(v) for v in kn.split(":")) for kn in os.environ.get("SHAPES", "4096:11008,11008:4096").split(",")]
for K, N in SHAPES:
    lins = [B.device_mx_linear(K, N, 64, seed=1 + i) for i in range(layers)]
    for M in [int(v) for v in os.environ.get("MS", "1,16").split(",")]:
        x = B.outlier_x(M, K)
        acts = [lin.quantize(x) for lin in lins]
        ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in lins]
        byts = N * K / 2 + N * K / 32 + N * 64 / 2 + N * 64 / 32 + M * K * (0.5 + 1 / 32) + 2 * M * N
        for v in variants:
            if v == "auto":
                os.environ.pop("SERQ_DEC_S", None)
            else:
                os.environ["SERQ_DEC_S"] = v
            def lin_all():
                for lin, a, y in zip(lins, acts, ys):
                    lin.gemm(a, y)
            def two_all():
                for lin, a, y in zip(lins, acts, ys):
                    lin.quantize(x, a)
                    lin.gemm(a, y)
            def fused_all():
                for lin, a, y in zip(lins, acts, ys):
                    lin.forward(x, a, y)
            r = {"K": K, "N": N, "M": M, "S": v}
            extra = int(os.environ.get("EXTRA_FLAGS", "0"))
            for name, fn in (("lin", lin_all), ("two", two_all), ("fused", fused_all)):
                _lib.call("serq_set_debug_flags", extra | (0 if name == "fused" else (1 << 23)))
                t = B.time_graph(B.graph_of(fn), None, n=10) / layers * 1e-3
                r[name + "_us"] = round(t * 1e6, 2)
                r[name + "_gbs"] = round(byts / t / 1e9)
            print(json.dumps(r), flush=True)
    del lins
    torch.cuda.empty_cache()
