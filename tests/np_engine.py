"""CPU engine for the sharded-truncation protocol (test infrastructure).

Implements the phase / slot interface of paper_1708_03340_b200.dist.GpuShardEngine
with the oracle's numpy node kernels, so the multi-rank protocol (who sends what,
when) runs under gloo on CPU exactly as it runs under NCCL on GPUs."""

import numpy as np
import torch

from oracle import htucker_oracle as orc
from paper_1708_03340_b200 import dist


class NumpyShardEngine:
    def __init__(self, x: "orc.HT", owned, ctl: "orc.Ctl", orth_ranks: dict):
        self.x, self.tr, self.ctl = x, x.tree, ctl
        self.owned = set(owned)
        nn = self.tr.n_nodes
        self.ko = orth_ranks
        self.orth, self.out = {}, {}
        kin = {t: x.rank(t) for t in range(1, nn)}
        # every slot exists up front (messages are received into them)
        self.R = {t: np.zeros((orth_ranks[t], kin[t])) for t in range(1, nn)}
        self.G = {t: np.zeros((orth_ranks[t], orth_ranks[t])) for t in range(1, nn)}
        self.EV = {t: np.zeros((orth_ranks[t], orth_ranks[t])) for t in range(1, nn)}
        self.lam = {t: np.zeros(orth_ranks[t]) for t in range(1, nn)}
        self.rk = np.ones(nn + 1, dtype=np.int32)

    def _order(self, nodes, bottom_up):
        levels = self.tr.levels()
        seq = [t for lev in (reversed(levels) if bottom_up else levels) for t in lev]
        s = set(nodes)
        return [t for t in seq if t in s]

    def phase(self, ph, nodes, out=None):
        tr = self.tr
        if ph == dist.ORTH:
            for t in self._order(nodes, True):
                if tr.is_leaf(t):
                    q, r = orc.qr_signfixed(self.x.U[t])
                    self.orth[t] = q
                    self.R[t][...] = r
                elif t == 0:
                    s1, s2 = tr.sons[0]
                    self.orth[0] = self.R[s1] @ self.x.root @ self.R[s2].T
                else:
                    s1, s2 = tr.sons[t]
                    b, r = orc.node_orth_inner(self.x.B[t], self.R[s1], self.R[s2])
                    self.orth[t] = b
                    self.R[t][...] = r
        elif ph == dist.GRAM:
            for t in self._order(nodes, False):
                if tr.is_leaf(t):
                    continue
                core, own = (self.orth[0][None], np.ones((1, 1))) if t == 0 else (self.orth[t], self.G[t])
                s1, s2 = tr.sons[t]
                g1, g2 = orc.node_gram_sons(core, own)
                self.G[s1][...] = g1
                self.G[s2][...] = g2
        elif ph == dist.EIG:
            for t in nodes:
                vec, lam = orc.eig_desc(self.G[t])
                self.EV[t][...] = vec
                self.lam[t][...] = lam
                self.rk[t] = orc.pick_rank(lam, self.ctl, t, tr.n_nodes - 1)
        elif ph == dist.PROJECT:
            r = out.ranks
            for t in nodes:
                if tr.is_leaf(t):
                    out.arrays[t][...] = torch.from_numpy(self.orth[t] @ self.EV[t][:, : r[t]])
                elif t == 0:
                    s1, s2 = tr.sons[0]
                    out.arrays[0][...] = torch.from_numpy(self.EV[s1][:, : r[s1]].T @ self.orth[0] @ self.EV[s2][:, : r[s2]])
                else:
                    s1, s2 = tr.sons[t]
                    out.arrays[t][...] = torch.from_numpy(orc.node_project_inner(
                        self.orth[t], self.EV[t][:, : r[t]], self.EV[s1][:, : r[s1]], self.EV[s2][:, : r[s2]]))

    def slot(self, kind, node):
        src = {dist.SLOT_R: self.R, dist.SLOT_G: self.G, dist.SLOT_EV: self.EV, dist.SLOT_LAM: self.lam}[kind]
        return torch.from_numpy(src[node]).view(-1)

    def ranks(self):
        return self.rk

    def allocate_out(self, ranks, nodes):
        sizes = {t: self.x.U[t].shape[0] for t in self.x.U}
        arrays = {}
        for t in nodes:
            node = self.tr
            if node.is_leaf(t):
                shape = (sizes[t], ranks[t])
            elif t == 0:
                shape = (ranks[node.sons[0][0]], ranks[node.sons[0][1]])
            else:
                s1, s2 = node.sons[t]
                shape = (ranks[t], ranks[s1], ranks[s2])
            arrays[t] = torch.zeros(shape, dtype=torch.float64)

        class Out:
            pass

        o = Out()
        o.ranks, o.arrays = ranks, arrays
        return o


class NumpyInnerEngine:
    """Phase / slot interface of dist.GpuInnerEngine with the oracle's Phi kernels."""

    def __init__(self, a: "orc.HT", c: "orc.HT"):
        self.a, self.c, self.tr = a, c, a.tree
        nn = self.tr.n_nodes
        self.phi = {t: np.zeros((a.rank(t), c.rank(t))) for t in range(1, nn)}
        self.res = torch.zeros(1, dtype=torch.float64)

    def phase(self, nodes):
        tr, s = self.tr, set(nodes)
        for lev in reversed(tr.levels()):
            for t in lev:
                if t not in s:
                    continue
                if tr.is_leaf(t):
                    self.phi[t][...] = self.a.U[t].T @ self.c.U[t]
                elif t == 0:
                    s1, s2 = tr.sons[0]
                    self.res[0] = float(np.sum((self.phi[s1].T @ self.a.root @ self.phi[s2]) * self.c.root))
                else:
                    s1, s2 = tr.sons[t]
                    self.phi[t][...] = orc.node_phi_inner(self.a.B[t], self.c.B[t], self.phi[s1], self.phi[s2])

    def slot(self, node):
        return torch.from_numpy(self.phi[node]).view(-1)

    def result(self):
        return self.res
