"""Per-call cost split for one request per call (C2 by default):
host enqueue cost of tts_decode_step with the device stalled, and device time
per call with the stream kept full (events around a run of calls)."""
import ctypes
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from synth import workload


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = workload.CONFIGS[name].with_(R=1)
    from paper_2509_00195_b200 import build
    build.build()
    from paper_2509_00195_b200.runner import Inputs, tts_config
    from paper_2509_00195_b200.tts import Context
    ctx = Context(tts_config(cfg, 1, num_pages=cfg.N * 80 + 64))
    lib, h, st = ctx.lib, ctx.h, ctx.stream
    inp = Inputs(cfg, ctx.device)
    kp, vp = inp.prompt_kv(0)
    q, k, v = inp.step(0, [0])
    out = torch.empty(cfg.L, 1, cfg.N, cfg.Hq, cfg.d, dtype=torch.float32, device=ctx.device)
    req = (ctypes.c_int32 * 1)(0)
    scale = ctypes.c_float(1.0 / math.sqrt(cfg.d))
    args = (ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(q.data_ptr()), scale,
            ctypes.c_void_p(out.data_ptr()), st)
    def prime():
        # same starting point for every measurement: fresh request, 64 tokens past the prompt
        lib.tts_block_table_release_request(h, 0, st)
        assert lib.tts_block_table_init_request(h, 0, cfg.N, cfg.prompt, kp.data_ptr(), vp.data_ptr(), st) == 0
        for _ in range(64):
            assert lib.tts_decode_step(h, 1, req, None, *args) == 0
        torch.cuda.synchronize()

    prime()
    if True:
        n = 48
        torch.cuda._sleep(int(2e9 // 1000 * 200))  # stall the stream ~ 0.2 s
        t0 = time.perf_counter()
        for _ in range(n):
            lib.tts_decode_step(h, 1, req, None, *args)
        host_us = (time.perf_counter() - t0) / n * 1e6
        torch.cuda.synchronize()
        prime()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n2 = 400
        e0.record()
        for _ in range(n2):
            lib.tts_decode_step(h, 1, req, None, *args)
        e1.record()
        torch.cuda.synchronize()
        dev_us = e0.elapsed_time(e1) / n2 * 1e3
        prime()
        ctx.tts_profile_begin()
        e0.record()
        for _ in range(n2):
            lib.tts_decode_step(h, 1, req, None, *args)
        e1.record()
        ms, cnt = ctx.tts_profile_end()
        torch.cuda.synchronize()
        print(f"{name}: with per-launch events: device {e0.elapsed_time(e1) / n2 * 1e3:.1f} us/call")
        attn_us = ms / max(cnt, 1) * 1e3
        # attention only (no append): same positions, kernel without a2
        qa = ctypes.c_void_p(q.data_ptr())
        prime()
        e0.record()
        for _ in range(n2):
            lib.tts_prefix_attn_decode(h, 0, cfg.L, 1, req, None, qa, scale, args[4], st)
        e1.record()
        torch.cuda.synchronize()
        attn_only_us = e0.elapsed_time(e1) / n2 * 1e3
    print(f"{name}: attention-only (no append) {attn_only_us:.1f} us/call")
    print(f"{name}: host enqueue {host_us:.1f} us/call, device {dev_us:.1f} us/call, attention {attn_us:.1f} us/call "
          f"(other {dev_us - attn_us:.1f})")


if __name__ == "__main__":
    main()
