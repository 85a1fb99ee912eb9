"""Per-shape timing of the conv kernels (fwd / dgrad / wgrad) on the GPU,
CUDA events around 20 launches after warm-up, for A/B decisions between kernel
variants (SN_CONV_PAIRS modes, TMA vs gather).  ResNet-50g b256 shapes.

    python tools/conv_bench.py [--pairs 0 1 2] [--ops fwd dgrad wgrad]
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [
    # N, C, H, W, K, k, stride, pad   (ResNet-50g b256, one of each distinct layer)
    (256, 64, 56, 56, 64, 3, 1, 1),
    (256, 64, 56, 56, 128, 3, 2, 1),
    (256, 128, 28, 28, 128, 3, 1, 1),
    (256, 128, 28, 28, 256, 3, 2, 1),
    (256, 256, 14, 14, 256, 3, 1, 1),
    (256, 256, 14, 14, 512, 3, 2, 1),
    (256, 512, 7, 7, 512, 3, 1, 1),
]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--halo", type=int, nargs="+", default=[1])
    ap.add_argument("--bn", type=int, nargs="+", default=[0], help="im2col tile width override (0 = policy)")
    ap.add_argument("--ops", nargs="+", default=["fwd", "dgrad", "wgrad"])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--shapes", type=int, nargs="+", default=None, help="indices into SHAPES")
    ap.add_argument("--shape", type=int, nargs=8, action="append", default=None,
                    metavar=("N", "C", "H", "W", "K", "k", "s", "p"), help="extra shape (repeatable)")
    args = ap.parse_args()
    import torch
    from paper_1801_04380_b200 import _native
    lib = _native.testing()
    lib.sn_test_conv.restype = ctypes.c_int
    lib.sn_test_conv.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.c_int]
    lib.sn_test_red_scratch_floats.restype = ctypes.c_longlong
    lib.sn_test_wgrad_splits.restype = ctypes.c_int
    dev = torch.device("cuda:0")
    shapes = [SHAPES[i] for i in (args.shapes if args.shapes is not None else range(len(SHAPES)))]
    if args.shape:
        shapes = ([SHAPES[i] for i in args.shapes] if args.shapes is not None else []) + [tuple(x) for x in args.shape]
    for shp in shapes:
        N, C, H, W, K, k, s, p = shp
        P = (H + 2 * p - k) // s + 1
        Q = (W + 2 * p - k) // s + 1
        shape = (ctypes.c_int * 11)(N, H, W, C, K, k, k, P, Q, s, p)
        x = torch.randn(N, H, W, C, device=dev)
        w = torch.randn(K, k, k, C, device=dev) * 0.05
        b = torch.randn(K, device=dev)
        y = torch.empty(N, P, Q, K, device=dev)
        dy = torch.randn(N, P, Q, K, device=dev)
        dx = torch.empty(N, H, W, C, device=dev)
        wt = torch.empty(K * k * k * C * 2, device=dev)
        dw = torch.empty(K, k, k, C, device=dev)
        db = torch.empty(K, device=dev)
        part = torch.empty(64 << 20, device=dev)
        red = torch.empty(int(lib.sn_test_red_scratch_floats(K)), device=dev)
        flops = 2.0 * N * P * Q * K * C * k * k
        for op in args.ops:
            if op == "fwd":
                ptrs = (ctypes.c_void_p * 4)(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr())
                call = lambda: lib.sn_test_conv(0, shape, ptrs, 0)
            elif op == "dgrad":
                ptrs = (ctypes.c_void_p * 4)(dy.data_ptr(), w.data_ptr(), wt.data_ptr(), dx.data_ptr())
                call = lambda: lib.sn_test_conv(1, shape, ptrs, 0)
            else:
                ptrs = (ctypes.c_void_p * 6)(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), db.data_ptr(),
                                             part.data_ptr(), red.data_ptr())
                call = lambda: lib.sn_test_conv(2, shape, ptrs, 0)
            line = f"{op:6s} N{N} C{C} {H}x{W} K{K} s{s}"
            for pm, hm, bn in [(pm, hm, bn) for hm in args.halo for pm in args.pairs for bn in args.bn]:
                lib.sn_test_set_conv_bn(bn)
                lib.sn_test_set_conv_pairs(pm)
                lib.sn_test_set_conv_halo(hm)
                lib.sn_test_set_sync(1)
                for _ in range(2):
                    assert call() == 0
                lib.sn_test_set_sync(0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.iters):
                    call()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.iters
                lib.sn_test_set_sync(1)
                tag = f"p{pm}h{hm}" + (f"b{bn}" if bn else "")
                line += f" | {tag}: {ms * 1e3:7.1f} us {flops / ms / 1e9:6.1f} TF/s"
            print(line, flush=True)
    lib.sn_test_set_conv_pairs(1)
    lib.sn_test_set_conv_bn(0)


if __name__ == "__main__":
    main()
