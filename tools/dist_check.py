"""Multi-process pipeline check (one stage per process) -- run under torchrun.

With RRFP_SAME_DEVICE=1 every rank uses cuda:0 (CUDA IPC between processes on
one GPU) so the IPC mailbox / peer-flag path can be exercised on a 1-GPU box.
Prints the last stage's loss and the single-process PP=1 loss of the same model.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    same = os.environ.get("RRFP_SAME_DEVICE") == "1"
    dev = 0 if same else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    from paper_2605_18750_b200.model import GPTConfig
    from paper_2605_18750_b200.distributed import DistPipeline
    cfg = GPTConfig(n_layer=4, d_model=256, n_head=2, d_ff=1024, vocab=512, seq=256)
    hint = sys.argv[1] if len(sys.argv) > 1 else "bf"
    tp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    chunks = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    mm = None
    split = "half" if len(sys.argv) > 4 and sys.argv[4] == "half" else "layer"   # stage cuts inside layers
    if len(sys.argv) > 4 and sys.argv[4] == "mm":   # config 4: ViT stage(s) + LLM stage(s)
        from paper_2605_18750_b200.model import MultimodalSpec
        vit = GPTConfig(n_layer=2, d_model=256, n_head=2, d_ff=512, vocab=0, seq=512, causal=False)
        cfg = GPTConfig(n_layer=2, d_model=256, n_head=2, d_ff=1024, vocab=512, seq=512)
        mm = MultimodalSpec(vit=vit, llm=cfg, vit_stages=world // 2, patch_tokens=128, d_patch=128,
                            max_images=4, image_seed=3)
    pipe = DistPipeline(cfg, 4, hint=hint, tp_size=tp, n_chunks=chunks, mm=mm, split=split)
    losses = []
    import time
    wd = float(os.environ.get("RRFP_WATCHDOG", "60"))
    for _ in range(2):
        t0 = time.time()
        loss = pipe.step(watchdog_secs=wd)
        print(f"[rank {rank}] step {time.time() - t0:.2f}s", file=sys.stderr, flush=True)
        dist.barrier()
        losses.append(None if loss is None else loss.item())
    ev, t0 = pipe.last_events
    n_exec = sum(1 for e in ev if e.kind == 0)
    off, rtt = pipe.calibrate_clocks(force=True)    # exercise the ping-pong even on one GPU
    pipe.calibrate_clocks()                         # the offsets actually applied (0 on one GPU)
    aligned = pipe.aligned_events()
    out = [None] * world   # (pipe is kept for its workload description)
    tp_err = pipe.comm.error() if pipe.comm else 0
    if os.environ.get("RRFP_REBUILD") == "1":
        # a second pipeline in the same processes (bench builds one per variant):
        # peer buffers must have been unmapped, warm-up must see fresh init
        wl = pipe.workload
        pipe.close()
        pipe = DistPipeline(cfg, 4, hint=hint, tp_size=tp, n_chunks=chunks, mm=mm, split=split)
        loss2 = pipe.step(watchdog_secs=wd)
        losses.append(None if loss2 is None else loss2.item())
        ev, t0 = pipe.last_events
    dist.all_gather_object(out, {"rank": rank, "losses": losses, "n_exec": n_exec, "tp_err": tp_err,
                                 "clock": [off, rtt], "events": aligned})
    pipe.close()
    if rank == 0:
        from paper_2605_18750_b200.pipeline import GpuPipeline
        ref = GpuPipeline(cfg, world // tp if mm else 1, 4, hint=hint, mm=mm)
        ref_loss = ref.step().item()
        ref.close()
        print(json.dumps({"ranks": out, "single_process_pp1_loss": ref_loss,
                          "workload": pipe.workload.to_json()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
