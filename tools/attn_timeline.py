"""Event timeline of one CTA of the attention forward (csrc/fmha_sm100.cu debug
hook, %clock64 cycles): producer waits, MMA waits (TMA data, P), softmax step
phases.   python tools/attn_timeline.py [--cta 0]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

NAMES = {0: "sm:wait_S", 1: "sm:S_ready", 2: "sm:S_loaded", 3: "sm:P_written", 4: "sm:P_arrived",
         5: "sm:max_done", 6: "sm:max_exchanged", 7: "sm:exp_chunk_done", 8: "sm:P_chunk_stored", 9: "sm:exp_start",
         10: "mma:wait_tile", 11: "mma:tile_ready", 12: "mma:wait_P", 13: "mma:P_ready",
         20: "tma:wait_slot", 21: "tma:slot_free",
         14: "mma:wait_dS", 15: "mma:dS_ready", 16: "mma:wait_dqbuf", 17: "mma:dqbuf_free", 18: "mma:grads_issued",
         30: "rd:wait_dQ", 31: "rd:dQ_ready", 32: "rd:reduce_issued"}
BWD_NAMES = {10: "mma:wait_stage", 11: "mma:stage_ready", 12: "mma:sd_free", 13: "mma:SD_issued",
             0: "ew:wait_S", 1: "ew:S_ready", 2: "ew:computed", 3: "ew:pds_free", 4: "ew:dS_stored", 5: "ew:S_loaded"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cta", type=int, nargs="+", default=[0, 112])
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--H", type=int, default=16)
    ap.add_argument("--bwd", action="store_true")
    a = ap.parse_args()
    from paper_2605_18750_b200 import _lib, kernels as K
    L = _lib.lib()
    T, H, D = a.T, a.H, a.H * 128
    qkv = torch.randn(T, 3 * D, device="cuda").to(torch.bfloat16)
    o = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, T, device="cuda")
    for _ in range(3):
        K.attn_fwd(qkv, o, lse, heads=H)
    if a.bwd:
        os.environ["RRFP_ATTN_DEBUG_BWD"] = "1"
        NAMES.update(BWD_NAMES)
        do = torch.randn(T, D, device="cuda").to(torch.bfloat16)
        dqkv = torch.empty(T, 3 * D, device="cuda", dtype=torch.bfloat16)
        ws = K.attn_bwd_workspace(T, H)
        for _ in range(3):
            K.attn_bwd(qkv, o, do, lse, dqkv, ws, heads=H)
    for cta in a.cta:
        buf = torch.zeros(4, 512, dtype=torch.int64, device="cuda")
        L.rrfp_attn_debug(C.c_void_p(buf.data_ptr()), cta)
        if a.bwd:
            K.attn_bwd(qkv, o, do, lse, dqkv, ws, heads=H)
        else:
            K.attn_fwd(qkv, o, lse, heads=H)
        torch.cuda.synchronize()
        L.rrfp_attn_debug(C.c_void_p(0), 0)
        ev = []
        for s in range(4):
            for x in buf[s].tolist():
                if x == 0:
                    break
                ev.append((x & 0xffffffffff, s, (x >> 56) & 0xff, (x >> 40) & 0xffff))
        ev.sort()
        t0 = ev[0][0]
        print(f"=== CTA {cta}: {len(ev)} events, span {ev[-1][0] - t0} cycles")
        for t, s, code, j in ev:
            lab = ('TMA MMA EW RD' if a.bwd else 'TMA MMA SM0 SM1').split()[s]
            print(f"{t - t0:8d}  {lab:4s} {NAMES.get(code, code):16s} {j}")


if __name__ == "__main__":
    main()
