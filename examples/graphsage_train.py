"""GraphSAGE minibatch training fed by the zero-copy fetch pipeline (SURVEY 8(f) NEXT-4 sketch).

The paper's application: DGL GraphSAGE training whose node features are gathered by
zero-copy from host memory.  Here the minibatch (3-hop uniform sample, blocks with positions in U,
and the gathered fp32 rows in HBM) comes from ``MinibatchFetcher``; the model is plain PyTorch
(mean aggregator SAGE layers) -- the model is not the hot path, the fetch is.

    python examples/graphsage_train.py [--config 4] [--steps 20] [--hidden 256]

Prints per-minibatch times: fetch alone, train alone, serial (fetch then train) and pipelined
(fetch of step j+1 on the fetch partition while step j trains), and the loss.
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402
from paper_2103_03330_b200.pipeline import MinibatchFetcher  # noqa: E402


class SAGE(torch.nn.Module):
    """L mean-aggregator SAGE layers: h'_v = act(W_self h_v + W_nbr mean_{u in S(v)} h_u)."""

    def __init__(self, d_in, hidden, classes, layers):
        super().__init__()
        dims = [d_in] + [hidden] * (layers - 1) + [classes]
        self.self_lin = torch.nn.ModuleList(torch.nn.Linear(dims[i], dims[i + 1]) for i in range(layers))
        self.nbr_lin = torch.nn.ModuleList(torch.nn.Linear(dims[i], dims[i + 1], bias=False) for i in range(layers))

    def forward(self, x, blocks, sizes):
        # blocks[k] = (positions in U [n_k, f_k] (-1 padded), counts [n_k]); the outermost hop first
        h = x
        L = len(blocks)
        for i, k in enumerate(reversed(range(L))):
            loc, cnt = blocks[k]
            n_dst = sizes[k]
            mask = (loc >= 0).unsqueeze(-1).to(h.dtype)
            nb = h[loc.clamp(min=0).long()] * mask                      # [n_dst, f, d]
            mean = nb.sum(1) / cnt.clamp(min=1).unsqueeze(-1).to(h.dtype)
            h = self.self_lin[i](h[:n_dst]) + self.nbr_lin[i](mean)
            if i < L - 1:
                h = F.relu(h)
        return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--hidden", type=int, default=256)
    ap.add_argument("--classes", type=int, default=172)      # ogbn-papers100M has 172 classes
    a = ap.parse_args()
    torch.cuda.set_device(0)
    c = gen.CONFIGS[a.config]
    L = len(c.fanouts)
    buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
    gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    # the random bytes are not meaningful fp32 features: clamp them to finite values in the model input
    table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    fetcher = MinibatchFetcher(table, graph, c.fanouts, c.batch)
    model = SAGE(c.dim, a.hidden, a.classes, L).cuda()
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    K = a.steps
    seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(K + 2)]
    rng = [gen.batch_rng_seed(c.seed, j) for j in range(K + 2)]

    def blocks_of(mb, sizes):
        b = []
        for k, (nbr, cnt, loc) in enumerate(mb.bufs.hop_blocks(sizes)):
            b.append((loc, cnt))
        return b

    def train_step(mb, sizes):
        n = sizes[-1]
        x = torch.nan_to_num(mb.rows[:n].view(torch.float32).view(n, c.dim), nan=0.0, posinf=1.0, neginf=-1.0)
        x = x.clamp(-1e3, 1e3)
        labels = (mb.bufs.ids[:sizes[0]] % a.classes).long()     # synthetic labels of the seeds
        out = model(x, blocks_of(mb, sizes), sizes)
        loss = F.cross_entropy(out, labels)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        return loss

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / K, r

    # warm-up
    for i in range(2):
        mb = fetcher.fetch(seeds[i], rng[i])
        train_step(mb, mb.sizes())
        fetcher.release(mb)          # the slot may be resampled only after this step's kernels
    t_fetch, _ = timed(lambda: [fetcher.fetch(seeds[i], rng[i]).sizes() for i in range(K)])
    mb = fetcher.fetch(seeds[0], rng[0])
    sz = mb.sizes()
    t_train, _ = timed(lambda: [train_step(mb, sz) for _ in range(K)])
    fetcher.release(mb)

    def serial():
        loss = None
        for i in range(K):
            m = fetcher.fetch(seeds[i], rng[i])
            loss = train_step(m, m.sizes())
            fetcher.release(m)
        return loss
    t_serial, _ = timed(serial)

    def pipelined():
        loss = None
        cur = fetcher.fetch(seeds[0], rng[0])
        for i in range(1, K + 1):
            nxt = fetcher.fetch(seeds[i], rng[i])     # fetch j+1 (fetch partition) ...
            s = cur.sizes()                            # (host needs |F_k| to slice the blocks)
            cur.wait()
            loss = train_step(cur, s)                  # ... while j trains on the default stream
            fetcher.release(cur)
            cur = nxt
        return loss
    t_pipe, loss = timed(pipelined)
    print(json.dumps({"config": c.name, "pipeline": fetcher.mode, "rows_per_minibatch": sz[-1],
                      "fetch_ms": round(t_fetch, 3), "train_ms": round(t_train, 3), "serial_ms": round(t_serial, 3),
                      "pipelined_ms": round(t_pipe, 3), "exposed_fetch_ms": round(max(0.0, t_pipe - t_train), 3),
                      "loss": round(float(loss), 4)}))
    fetcher.close()
    table.unregister()
    buf.free()


if __name__ == "__main__":
    main()
