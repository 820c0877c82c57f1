"""Convergence vs batch size (the paper's batch-size
study, PAPER.md:186-199 / Fig. 1b: larger minibatches run faster per example
but "updates to weights accumulate", so more examples are needed to converge).

Synthetic bigram-structured corpus (synth.bigram_corpus: every word has
`branching` successors), windows at i.i.d. positions of the training part,
uniformly corrupted centres.  For each batch size B the same example sequence
is consumed B at a time through PolyglotModel.train_step (the fused sm_100a
step); every `--val-every` examples the validation loss -- the mean hinge
max(0, 1 - s + s') over 1000 held-out windows with fixed corrupt centres,
scores from pg_score -- is checked against the target.  Reported per B: the
examples, steps and device time (CUDA events around the training steps only)
until the target is reached.  Output: one JSON document (stdout, and --out).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1404_1521_b200 as pg
import synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vocab", type=int, default=10_000)
    ap.add_argument("--dim", type=int, default=64)
    ap.add_argument("--window", type=int, default=5)
    ap.add_argument("--hidden", type=int, default=32)
    ap.add_argument("--branching", type=int, default=4)
    ap.add_argument("--batches", default="16,32,64,128,256,512")
    ap.add_argument("--lrs", default="0.1,0.3,1,3", help="lr grid; every B reports its best")
    ap.add_argument("--lr-scaling", choices=["const", "linear"], default="const",
                    help="linear: lr x B per step, i.e. the summed-loss reading of G4 (PAPER.md:197-198)")
    ap.add_argument("--target", type=float, default=0.05)
    ap.add_argument("--max-examples", type=int, default=8_000_000)
    ap.add_argument("--val-every", type=int, default=32_768, help="examples between validations")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    V, d, n, h = a.vocab, a.dim, a.window, a.hidden
    dev = torch.device("cuda")
    t0 = time.time()
    corpus_len = 4_000_000
    toks = synth.bigram_corpus(V, corpus_len + 100_000, a.seed, a.branching)
    tr_idx, tr_corr = synth.corpus_batch(toks, V, n, a.max_examples, a.seed, 0, 0, corpus_len)
    va_idx, va_corr = synth.corpus_batch(toks, V, n, 1000, a.seed, 1, corpus_len, toks.shape[0])
    va_bad = va_idx.copy()
    va_bad[:, n // 2] = va_corr
    d_idx, d_corr = torch.from_numpy(tr_idx).to(dev), torch.from_numpy(tr_corr).to(dev)
    d_va, d_vb = torch.from_numpy(va_idx).to(dev), torch.from_numpy(va_bad).to(dev)
    gen_s = time.time() - t0
    stream = torch.cuda.Stream()
    results = {}
    for B, lr0 in [(int(x), float(y)) for x in a.batches.split(",") for y in a.lrs.split(",")]:
        m = pg.PolyglotModel(V, d, n, h, seed=a.seed, stream=stream)
        lr = lr0 * B if a.lr_scaling == "linear" else lr0
        m.reserve(B)
        s_true = torch.empty(1000, device=dev)
        s_bad = torch.empty(1000, device=dev)

        def val_loss():
            with torch.cuda.stream(stream):
                m.score(d_va, s_true)
                m.score(d_vb, s_bad)
                return float(torch.clamp(1.0 - s_true + s_bad, min=0.0).mean().item())

        curve = [(0, val_loss())]
        steps_per_val = max(1, a.val_every // B)
        max_steps = a.max_examples // B
        step, dev_ms, reached = 0, 0.0, None
        while step < max_steps and reached is None:
            k = min(steps_per_val, max_steps - step)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                ev0.record(stream)
                for t in range(step, step + k):
                    m.train_step(d_idx[t * B:(t + 1) * B], d_corr[t * B:(t + 1) * B], lr, loss_out=None)
                ev1.record(stream)
            stream.synchronize()
            dev_ms += ev0.elapsed_time(ev1)
            step += k
            vl = val_loss()
            curve.append((step * B, vl))
            if vl < a.target:
                reached = {"examples": step * B, "steps": step, "device_s": dev_ms / 1e3}
        m.sync()
        m.close()
        results.setdefault(str(B), {})[str(lr0)] = {"lr": lr, "reached": reached, "final_val_loss": curve[-1][1],
                           "examples_per_device_s": step * B / (dev_ms / 1e3),
                           "curve": curve[:: max(1, len(curve) // 40)] + ([curve[-1]] if len(curve) > 40 else [])}
        print(f"B={B:4d} lr={lr:g} reached={reached} final={curve[-1][1]:.4f}", file=sys.stderr, flush=True)
    best = {}
    for B, runs in results.items():
        ok = [(r["reached"]["device_s"], k) for k, r in runs.items() if r["reached"]]
        best[B] = dict(runs[min(ok)[1]]["reached"], lr=runs[min(ok)[1]]["lr"]) if ok else None
    doc = {"study": "convergence vs batch size (SURVEY.md 8(f) NEXT-1)",
           "model": {"vocab": V, "dim": d, "window": n, "hidden": h},
           "corpus": f"bigram Markov chain, {a.branching} successors per word, {corpus_len} training tokens, "
                     f"windows at i.i.d. positions, uniform corrupt centres, seed {a.seed}",
           "lr_grid": a.lrs, "lr_scaling": a.lr_scaling, "best_per_batch": best,
           "loss": "mean hinge over the batch (reading G4); lr_scaling=linear is the summed-loss reading",
           "target_val_loss": a.target, "validation": "1000 held-out windows, fixed corrupt centres, pg_score",
           "time": "device time of the training steps (CUDA events), validation excluded",
           "gpu": torch.cuda.get_device_name(0), "input_generation_s": gen_s, "results": results}
    js = json.dumps(doc)
    print(js)
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
