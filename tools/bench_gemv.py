"""Time the grouped decode GEMV (K5) at the 8B decode shapes, 4 modules x
M rows each, CUDA-graph replay over all layers' weights (working set >> L2).

    python tools/bench_gemv.py [M]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2602_12029_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
TC = len(sys.argv) > 2 and sys.argv[2] == "tc"  # psk_gemv_tc (tcgen05) instead of psk_gemv
import ctypes  # noqa: E402
lib = _lib.load()
N_MOD, L = 4, 8
d, ffn, vocab = 4096, 14336, 128256
shapes = {"qkv": (6144, d, 1), "o": (d, d, 2), "gate_up": (2 * ffn, d, 3), "down": (d, ffn, 2),
          "head": (vocab, d, 1)}
peak = 6548.5
for name, (N, K, epi) in shapes.items():
    layers = 1 if name == "head" else L
    W = [[torch.empty(N, K, dtype=torch.bfloat16, device="cuda") for _ in range(N_MOD)]
         for _ in range(layers)]
    for lw in W:
        for w in lw:
            _lib.check(lib.psk_init_normal_bf16(w.data_ptr(), w.numel(), 5, 0.02, 0))
    ptrs = [torch.tensor([w.data_ptr() for w in lw], dtype=torch.int64, device="cuda") for lw in W]
    R = N_MOD * M
    x = torch.randn(R, K, device="cuda").to(torch.bfloat16)
    mrs = torch.tensor([i * M for i in range(N_MOD + 1)], dtype=torch.int32, device="cuda")
    out = torch.zeros(R, N if epi != 3 else N // 2, dtype=torch.float32 if epi in (1, 2) else torch.bfloat16,
                      device="cuda")
    st = torch.cuda.Stream()
    reps = 4 * layers if name != "head" else 8

    hps = [(ctypes.c_void_p * N_MOD)(*[w.data_ptr() for w in lw]) for lw in W]
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_gemv_tc_workspace(ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value, dtype=torch.uint8, device="cuda")

    def launch(i):
        if TC:
            _lib.check(lib.psk_gemv_tc(x.data_ptr(), R, K, hps[i % layers], mrs.data_ptr(), N_MOD, M, N,
                                       epi, out.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream))
        else:
            _lib.check(lib.psk_gemv(x.data_ptr(), R, K, ptrs[i % layers].data_ptr(), mrs.data_ptr(), N_MOD, M, N,
                                    epi, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    with torch.cuda.stream(st):
        for i in range(3):
            launch(i)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(reps):
                launch(i)
        g.replay()
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g.replay()
        b.record(st)
    b.synchronize()
    dt = a.elapsed_time(b) / 1e3 / reps
    nbytes = N_MOD * N * K * 2
    print(f"{'tc ' if TC else ''}{name:8s} N={N:6d} K={K:5d} M={M}: {dt * 1e6:8.1f} us  {nbytes / dt / 1e9:7.1f} GB/s "
          f"({nbytes / dt / 1e9 / peak:.3f} of {peak})")
    del W, ptrs
    torch.cuda.empty_cache()
