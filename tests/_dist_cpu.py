"""Test-only CPU engine for the partitioned BFS orchestration
(paper_1701_01170_b200/dist.py).  It implements the same per-rank steps as
the device engine (csrc/gfx_dist.cu) with numpy, so the host-side
orchestration -- direction decisions on global counts, all_to_all of
(dst, src) pairs, all_gather of frontier bitmaps -- can be exercised across
real gloo processes on a machine without a GPU.  Never used by the product."""
import numpy as np
import torch

UNV = np.iinfo(np.int32).max


class CpuEngine:
    def __init__(self, row, col, n, m, P, r):
        self.P, self.r, self.n, self.m = P, r, int(n), int(m)
        self.device = torch.device("cpu")
        owned = np.arange(r, n, P, dtype=np.int64)
        self.nl = len(owned)
        deg = row[owned + 1] - row[owned]
        self.lrow = np.zeros(self.nl + 1, dtype=np.int64)
        np.cumsum(deg, out=self.lrow[1:])
        self.lcol = np.concatenate([col[row[v]:row[v + 1]] for v in owned]).astype(np.int64) \
            if self.nl and self.lrow[-1] else np.zeros(0, dtype=np.int64)
        nmax = (n + P - 1) // P
        self.wmax = (nmax + 31) // 32
        self.send = torch.zeros(n + 64, dtype=torch.int64)
        self.recv = torch.zeros(n + 64, dtype=torch.int64)
        self.front_local = torch.zeros(self.wmax, dtype=torch.int32)
        self.gathered = torch.zeros(P * self.wmax, dtype=torch.int32)
        self.counts = torch.zeros(2 * P, dtype=torch.int64)
        self.send_counts, self.recv_counts = self.counts[:P], self.counts[P:]
        self.stats = torch.zeros(8, dtype=torch.int64)

    def reset(self, source):
        self.labels = np.full(self.nl, UNV, dtype=np.int64)
        self.preds = np.full(self.nl, -1, dtype=np.int64)
        self.frontier = np.zeros(0, dtype=np.int64)
        if source % self.P == self.r:
            l = source // self.P
            self.labels[l] = 0
            self.frontier = np.array([l], dtype=np.int64)
        return len(self.frontier)

    def _claim(self, ls, srcs, depth):
        """first occurrence of each unvisited local id wins"""
        ok = self.labels[ls] == UNV
        ls, srcs = ls[ok], srcs[ok]
        ls, first = np.unique(ls, return_index=True)
        self.labels[ls] = depth
        self.preds[ls] = srcs[first]
        return ls

    def push_expand(self, depth):
        F = self.frontier
        deg = self.lrow[F + 1] - self.lrow[F]
        src = np.repeat(F * self.P + self.r, deg)
        dst = np.concatenate([self.lcol[self.lrow[l]:self.lrow[l + 1]] for l in F]) \
            if len(F) else np.zeros(0, dtype=np.int64)
        own = dst % self.P == self.r
        self.local_new = self._claim(dst[own] // self.P, src[own], depth)
        rd, rs = dst[~own], src[~own]
        rd, first = np.unique(rd, return_index=True)
        rs = rs[first]
        counts, pairs = [], []
        for o in range(self.P):
            sel = rd % self.P == o
            if o == self.r:
                counts.append(0)
                continue
            counts.append(int(sel.sum()))
            pairs.append((rd[sel] << 32) | rs[sel])
        flat = np.concatenate(pairs) if pairs else np.zeros(0, dtype=np.int64)
        self.send[: len(flat)] = torch.from_numpy(flat)
        self.send_counts[:] = torch.tensor(counts, dtype=torch.int64)
        self.stats[:] = torch.tensor([0, int(deg.sum()), 0, 0] * 2)

    def push_claim(self, nrecv, depth):
        x = self.recv[:nrecv].numpy()
        d, s = x >> 32, x & 0xFFFFFFFF
        got = self._claim(d // self.P, s, depth)
        self.frontier = np.concatenate([self.local_new, got])
        self.stats[0] = self.stats[4] = len(self.frontier)

    def pull_prepare(self):
        bits = np.zeros(self.wmax * 32, dtype=bool)
        bits[self.frontier] = True
        self.front_local[:] = _pack(bits)

    def pull(self, depth):
        g = self.gathered.numpy().view(np.uint32)
        found, par = [], []
        probes = cands = 0
        for u in np.flatnonzero(self.labels == UNV):
            nb = self.lcol[self.lrow[u]:self.lrow[u + 1]]
            if len(nb) == 0:
                continue
            cands += 1
            for k, s in enumerate(nb):
                lo = s // self.P
                if (g[(s % self.P) * self.wmax + (lo >> 5)] >> (lo & 31)) & 1:
                    found.append(u)
                    par.append(s)
                    probes += k + 1
                    break
            else:
                probes += len(nb)
        found = np.array(found, dtype=np.int64)
        self.labels[found] = depth
        self.preds[found] = np.array(par, dtype=np.int64)
        self.frontier = found
        self.stats[:] = torch.tensor([len(found), 0, probes, cands] * 2)

    def commit(self, nf_local):
        assert nf_local == len(self.frontier)


def _pack(bits):
    words = np.zeros(len(bits) // 32, dtype=np.uint32)
    idx = np.flatnonzero(bits)
    np.bitwise_or.at(words, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    return torch.from_numpy(words.view(np.int32))


class CpuSsspEngine:
    """Test-only numpy engine with the per-rank steps of csrc/gfx_dsssp.cu
    (relax with owned/remote split and the monotone sent-offer filter,
    (d, dist<<32|pred) messages of 2 words, owner-side min, near/far split,
    stale-dropping re-split), so sssp_partitioned's host orchestration can run
    across real gloo processes without a GPU."""

    INF = np.iinfo(np.int64).max

    def __init__(self, row, col, w, n, P, r):
        self.P, self.r, self.n = P, r, int(n)
        self.device = torch.device("cpu")
        owned = np.arange(r, n, P, dtype=np.int64)
        self.nl = len(owned)
        deg = row[owned + 1] - row[owned]
        self.lrow = np.zeros(self.nl + 1, dtype=np.int64)
        np.cumsum(deg, out=self.lrow[1:])
        idx = np.concatenate([np.arange(row[v], row[v + 1]) for v in owned]) \
            if self.nl and self.lrow[-1] else np.zeros(0, dtype=np.int64)
        self.lcol = col[idx].astype(np.int64)
        self.lw = w[idx].astype(np.int64)
        ml = len(self.lcol)
        self.send = torch.zeros(2 * (min(ml, n) + 64), dtype=torch.int64)
        self.recv = torch.zeros(2 * (max(P - 1, 1) * self.nl + 64), dtype=torch.int64)
        self.counts = torch.zeros(2 * P, dtype=torch.int64)
        self.send_counts, self.recv_counts = self.counts[:P], self.counts[P:]
        self.stats = torch.zeros(8, dtype=torch.int64)

    def reset(self, source):
        self.dist = np.full(self.nl, self.INF, dtype=np.int64)
        self.pred = np.full(self.nl, -1, dtype=np.int64)
        self.sent_best = np.full(self.n, self.INF, dtype=np.int64)
        self.near = np.zeros(0, dtype=np.int64)
        self.far = np.zeros(0, dtype=np.int64)
        self.far_key = np.zeros(0, dtype=np.int64)
        if source % self.P == self.r:
            l = source // self.P
            self.dist[l] = 0
            self.near = np.array([l], dtype=np.int64)
        return len(self.near)

    def _offer(self, ls, nd, src):
        """owner-side relax: improved local ids, once (sorted unique)"""
        order = np.lexsort((src, nd, ls))
        ls, nd, src = ls[order], nd[order], src[order]
        first = np.ones(len(ls), dtype=bool)
        first[1:] = ls[1:] != ls[:-1]
        ls, nd, src = ls[first], nd[first], src[first]
        better = nd < self.dist[ls]
        ls, nd, src = ls[better], nd[better], src[better]
        self.dist[ls] = nd
        self.pred[ls] = src
        return ls

    def relax(self):
        F = self.near
        deg = self.lrow[F + 1] - self.lrow[F]
        src = np.repeat(F * self.P + self.r, deg)
        sd = np.repeat(self.dist[F], deg)
        sl = np.concatenate([np.arange(self.lrow[l], self.lrow[l + 1]) for l in F]) \
            if len(F) else np.zeros(0, dtype=np.int64)
        d, nd = self.lcol[sl], sd + self.lw[sl]
        own = d % self.P == self.r
        self.touched = self._offer(d[own] // self.P, nd[own], src[own])
        rd, rn, rs = d[~own], nd[~own], src[~own]
        order = np.lexsort((rs, rn, rd))
        rd, rn, rs = rd[order], rn[order], rs[order]
        first = np.ones(len(rd), dtype=bool)
        first[1:] = rd[1:] != rd[:-1]
        rd, rn, rs = rd[first], rn[first], rs[first]
        keep = rn < self.sent_best[rd]
        rd, rn, rs = rd[keep], rn[keep], rs[keep]
        self.sent_best[rd] = rn
        words, counts = [], []
        for o in range(self.P):
            sel = rd % self.P == o
            counts.append(2 * int(sel.sum()))
            if sel.any():
                msg = np.empty(2 * int(sel.sum()), dtype=np.int64)
                msg[0::2] = rd[sel]
                msg[1::2] = (rn[sel] << 32) | rs[sel]
                words.append(msg)
        flat = np.concatenate(words) if words else np.zeros(0, dtype=np.int64)
        self.send[: len(flat)] = torch.from_numpy(flat)
        self.send_counts[:] = torch.tensor(counts, dtype=torch.int64)
        self.slots = int(deg.sum())

    def apply(self, nrecv_words):
        x = self.recv[:nrecv_words].numpy()
        d, key = x[0::2], x[1::2]
        got = self._offer(d // self.P, key >> 32, key & 0xFFFFFFFF)
        self.touched = np.union1d(self.touched, got)

    def _stats(self, slots, touched):
        self.stats[:] = torch.tensor([len(self.near), len(self.far), slots, touched] * 2)

    def split(self, threshold):
        t = self.touched
        keys = self.dist[t]
        near = keys < threshold
        self.near = t[near]
        self.far = np.concatenate([self.far, t[~near]])
        self.far_key = np.concatenate([self.far_key, keys[~near]])
        self._stats(self.slots, len(t))

    def refar(self, threshold, split, far_local):
        assert far_local == len(self.far)
        fresh = self.dist[self.far] == self.far_key
        items, keys = self.far[fresh], self.far_key[fresh]
        near = (keys < threshold) if split else np.zeros(len(items), dtype=bool)
        if split:
            self.near = items[near]
        self.far, self.far_key = items[~near], keys[~near]
        self._stats(0, 0)

    def result(self):
        return self.dist, self.pred
