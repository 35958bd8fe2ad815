"""Balanced dimension trees (mirror of the reference ``htucker.tree``).

Same node numbering as the reference (tree.py:55-101): breadth-first ids,
root 0, a node over modes ``{mu..nu}`` splits at ``(mu + nu - 1) // 2``, so the
depth is ``ceil(log2 d)`` and there are ``2d - 1`` nodes.  The C++ driver
(csrc/driver.cu) builds the identical tree from ``d``; this host copy serves the
Python API (levels, sons, leaf lookup) and the multi-GPU shard map.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TreeNode:
    index: int
    interval: tuple
    father: int | None
    sons: tuple | None
    level: int

    @property
    def is_leaf(self) -> bool:
        return self.sons is None

    @property
    def is_root(self) -> bool:
        return self.father is None

    @property
    def dims(self) -> range:
        return range(self.interval[0], self.interval[1] + 1)

    @property
    def dim(self) -> int:
        if not self.is_leaf:
            raise ValueError(f"node {self.index} is not a leaf")
        return self.interval[0]


class DimensionTree:
    """Balanced dimension tree for ``d >= 2`` (reference tree.py:60-154)."""

    def __init__(self, d: int):
        if d < 2:
            raise ValueError(f"tensor dimension must be >= 2, got {d}")
        self.d = int(d)
        order = [((1, self.d), None, 0)]
        info = []
        head = 0
        while head < len(order):
            (mu, nu), father, level = order[head]
            info.append([(mu, nu), father, level, None])
            if mu != nu:
                cut = (mu + nu - 1) // 2
                order.append(((mu, cut), head, level + 1))
                order.append(((cut + 1, nu), head, level + 1))
            head += 1
        sons = {}
        for idx, (_, father, _, _) in enumerate(info):
            if father is not None:
                sons.setdefault(father, []).append(idx)
        self.nodes = [TreeNode(i, iv, fa, tuple(sons[i]) if i in sons else None, lev)
                      for i, (iv, fa, lev, _) in enumerate(info)]
        self.depth = max(n.level for n in self.nodes)
        self._levels = [[] for _ in range(self.depth + 1)]
        for n in self.nodes:
            self._levels[n.level].append(n.index)
        self._leaf_of_dim = {n.dim: n.index for n in self.nodes if n.is_leaf}

    def __len__(self) -> int:
        return len(self.nodes)

    @property
    def root(self) -> TreeNode:
        return self.nodes[0]

    def node(self, index: int) -> TreeNode:
        return self.nodes[index]

    def sons(self, index: int):
        pair = self.nodes[index].sons
        if pair is None:
            raise ValueError(f"node {index} is a leaf")
        return self.nodes[pair[0]], self.nodes[pair[1]]

    def leaf_for_dim(self, mu: int) -> TreeNode:
        return self.nodes[self._leaf_of_dim[mu]]

    @property
    def leaves(self):
        return [self.leaf_for_dim(mu) for mu in range(1, self.d + 1)]

    @property
    def inner_nodes(self):
        return [n for n in self.nodes if not n.is_leaf and not n.is_root]

    @property
    def non_root(self):
        return self.nodes[1:]

    def levels_top_down(self):
        return [list(level) for level in self._levels]

    def edges(self):
        return [(n.father, n.index) for n in self.nodes if n.father is not None]

    def subtree(self, index: int):
        """Node ids of the subtree rooted at ``index`` (used by the shard map)."""
        out, stack = [], [index]
        while stack:
            t = stack.pop()
            out.append(t)
            if self.nodes[t].sons is not None:
                stack.extend(self.nodes[t].sons)
        return sorted(out)

    def __eq__(self, other) -> bool:
        return isinstance(other, DimensionTree) and other.d == self.d

    def __hash__(self) -> int:
        return hash(("DimensionTree", self.d))

    def __repr__(self) -> str:
        return f"DimensionTree(d={self.d}, nodes={len(self.nodes)}, depth={self.depth})"


_cache: dict = {}


def build_balanced_tree(d: int) -> DimensionTree:
    if d not in _cache:
        _cache[d] = DimensionTree(d)
    return _cache[d]


def nodes_at_level(tree: DimensionTree, level: int):
    if level < 0 or level > tree.depth:
        raise ValueError(f"level {level} out of range [0, {tree.depth}]")
    return list(tree.levels_top_down()[level])
