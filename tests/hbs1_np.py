"""Test helper: read an HBS1 file (hbs.cpp:681-808 layout)
into numpy and run the telescoping solve split by subtrees on the host.

This is test infrastructure: it restates the subtree partition of
paper_2108_07205_b200/csrc/sweep.cu (hbs_shard) so the exchange protocol of
paper_2108_07205_b200/parallel.py can be exercised over gloo without a GPU.
"""
import struct

import numpy as np


class Node:
    pass


def read_hbs1(path):
    buf = open(path, "rb").read()
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from("<" + fmt, buf, off)
        off += struct.calcsize("<" + fmt)
        return v

    def idx():
        (n,) = take("q")
        return np.array(take(f"{n}q"), dtype=np.int64) if n else np.zeros(0, np.int64)

    def mat():
        r, c = take("qq")
        a = np.array(take(f"{r * c}d"), dtype=np.float64) if r * c else np.zeros(0)
        return a.reshape((r, c), order="F")

    assert buf[:4] == b"HBS1"
    off = 4
    (version,) = take("I")
    assert version == 1
    (has_inv,) = take("B")
    n, leaf, eps, mbd, count = take("qqdqq")
    nodes = []
    for _ in range(count):
        nd = Node()
        nd.begin, nd.end, nd.parent, nd.left, nd.right = take("qqqqq")
        (nd.depth,) = take("i")
        (nd.k,) = take("q")
        nd.row_skel, nd.col_skel = idx(), idx()
        nd.u, nd.v, nd.d, nd.b_sib, nd.dhat, nd.e, nd.f, nd.g = (mat() for _ in range(8))
        nodes.append(nd)
    root_g = mat()
    return {"n": n, "has_inverse": bool(has_inv), "nodes": nodes, "root_g": root_g}


class HostShardExecutor:
    """Rank p of G: the same subtree split as hbs_shard (sweep.cu), in numpy."""

    def __init__(self, op, G, p):
        nodes = op["nodes"]
        g = G.bit_length() - 1
        assert 1 << g == G
        self.op, self.G, self.p, self.g = op, G, p, g
        self.roots = [i for i, nd in enumerate(nodes) if nd.depth == g]
        assert len(self.roots) == G
        owner = [-1] * len(nodes)
        for q, r in enumerate(self.roots):
            owner[r] = q
        for i, nd in enumerate(nodes):
            if nd.depth > g:
                owner[i] = owner[nd.parent]
        self.owner = owner
        sr = nodes[self.roots[p]]
        self.row0, self.row1 = 2 * sr.begin, 2 * sr.end
        self.kmax = max(nodes[r].k for r in self.roots) if g > 0 else 0
        self.hat, self.pp, self.inc = {}, {}, {}

    def _up(self, i, b):
        nd = self.op["nodes"][i]
        if nd.left < 0:
            bi = b[2 * nd.begin - self.row0: 2 * nd.end - self.row0]
        else:
            bi = np.vstack([self.hat[nd.left], self.hat[nd.right]])
        self.hat[i] = nd.f @ bi
        self.pp[i] = nd.g @ bi

    def up(self, b_local):
        nodes = self.op["nodes"]
        mine = [i for i in range(1, len(nodes)) if self.owner[i] == self.p]
        for d in range(max(nd.depth for nd in nodes), self.g - 1, -1):
            for i in mine:
                if nodes[i].depth == d:
                    self._up(i, b_local)
        nrhs = b_local.shape[1]
        out = np.zeros((self.kmax, nrhs))
        if self.g > 0:
            r = self.roots[self.p]
            out[: nodes[r].k] = self.hat[r]
        return out

    def down(self, hats, nrhs):
        nodes = self.op["nodes"]
        if self.g > 0:
            for q, r in enumerate(self.roots):
                if q != self.p:
                    self.hat[r] = np.asarray(hats[q])[: nodes[r].k]
        for d in range(self.g - 1, 0, -1):  # top up-levels (redundant)
            for i, nd in enumerate(nodes):
                if i and nd.depth == d:
                    self._up(i, None)
        root = nodes[0]
        if root.left < 0:
            raise ValueError("single-leaf tree")
        y = self.op["root_g"] @ np.vstack([self.hat[root.left], self.hat[root.right]])
        kl = nodes[root.left].k
        self.inc[root.left], self.inc[root.right] = y[:kl], y[kl:]
        x = np.zeros((self.row1 - self.row0, nrhs))
        for d in range(1, max(nd.depth for nd in nodes) + 1):
            for i, nd in enumerate(nodes):
                if not i or nd.depth != d:
                    continue
                if d >= self.g and self.owner[i] != self.p:
                    continue
                z = nd.e @ self.inc[i] + self.pp[i]
                if nd.left < 0:
                    x[2 * nd.begin - self.row0: 2 * nd.end - self.row0] = z
                else:
                    kl = nodes[nd.left].k
                    self.inc[nd.left], self.inc[nd.right] = z[:kl], z[kl:]
        return x
