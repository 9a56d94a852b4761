"""System ablation with a real backward pass (paper E10; SURVEY
NEXT-2): per-iteration time of forward + backward + ACP-SGD aggregation on
synthetic inputs, random-init weights, for

  none      forward + backward only (no gradient exchange): the floor
  naive     backward, then the whole ACP step (compress, all-reduce, decode)
  wfbp      one tensor per bucket, compressed + all-reduced from grad hooks
  wfbp_tf   the paper's buckets (25 MiB x compression rate) from grad hooks

One process per GPU (torchrun for N > 1); max over ranks of the CUDA-event
time. Prints one JSON line per mode (rank 0).

  python scripts/wfbp_bench.py --model bert-large --rank 4
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/wfbp_bench.py --model resnet152
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_model(name, batch):
    import torch
    if name == "bert-large" or name == "bert-base":
        from transformers import BertConfig, BertForPreTraining
        cfg = BertConfig() if name == "bert-base" else BertConfig(
            hidden_size=1024, num_hidden_layers=24, num_attention_heads=16, intermediate_size=4096)
        model = BertForPreTraining(cfg).cuda()
        seq = 128
        ids = torch.randint(0, cfg.vocab_size, (batch, seq), device="cuda")
        labels = torch.randint(0, cfg.vocab_size, (batch, seq), device="cuda")
        nsp = torch.randint(0, 2, (batch,), device="cuda")

        def loss_fn():
            out = model(input_ids=ids, labels=labels, next_sentence_label=nsp)
            return out.loss
        return model, loss_fn
    import torchvision
    model = getattr(torchvision.models, name.replace("-", ""))().cuda()
    x = torch.randn(batch, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (batch,), device="cuda")
    crit = torch.nn.CrossEntropyLoss()

    def loss_fn():
        return crit(model(x), y)
    return model, loss_fn


def main():
    import torch
    import torch.distributed as dist
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bert-large")
    ap.add_argument("--rank", type=int, default=4)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--amp", action="store_true", help="bf16 autocast forward/backward")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2306_08881_b200 import nccl_comm_from_group
        comm = nccl_comm_from_group()
    from paper_2306_08881_b200.wfbp import Wfbp
    batch = args.batch or (32 if args.model.startswith("bert") else 64)
    model, loss_fn = build_model(args.model, batch)
    nparam = sum(p.numel() for p in model.parameters())

    def run(mode):
        wf = None
        if mode != "none":
            wf = Wfbp(model, args.rank, world_size=world, nccl_comm=comm, seed=3,
                      bucket_bytes=0 if mode == "wfbp" else 25 * 2 ** 20, overlap=mode != "naive")
        times = []
        for it in range(args.warmup + args.steps):
            if wf is not None:
                wf.begin(it % 2)
            else:
                model.zero_grad(set_to_none=False)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=args.amp):
                loss = loss_fn()
            loss.backward()
            if wf is not None:
                wf.end()
            e1.record()
            torch.cuda.synchronize()
            if it >= args.warmup:
                times.append(e0.elapsed_time(e1))
        ms = sum(times) / len(times)
        if world > 1:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        nb = wf.num_buckets(0) if wf is not None else 0
        if wf is not None:
            wf.close()
            for p in model.parameters():
                p.grad = None
        return ms, nb

    res = {}
    for mode in ("none", "naive", "wfbp", "wfbp_tf"):
        res[mode] = run(mode)
    if rank == 0:
        base = res["none"][0]
        for mode, (ms, nb) in res.items():
            print(json.dumps({"model": args.model, "rank": args.rank, "n_gpus": world, "batch": batch,
                              "amp": args.amp, "params": nparam, "mode": mode, "ms_per_iter": ms,
                              "buckets_P": nb, "overhead_vs_none_ms": ms - base}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
