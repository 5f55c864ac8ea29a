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
