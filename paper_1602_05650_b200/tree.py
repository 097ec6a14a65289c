"""Octree Stokeslet summation (the reference's TreeSummation backend,
system.py:108-224) with the evaluation on the device (sf_tree_stokeslet).

The host builds the octree TOPOLOGY from the source positions with the
reference's octant split (system.py:112-140) -- one pass per geometry,
cached -- and permutes the sources so every node owns a contiguous range.
Every call computes the node moments from the strengths, traverses the tree
with the reference's opening test and subtracts the same-group partials, all
on the device.
"""

import ctypes
import hashlib

import numpy as np

from . import _native


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


def build_topology(pts, leaf_size):
    """Octree of the points (system.py:112-140): returns (perm, nbeg, nend,
    first_child, nchild) with each node's points perm[nbeg:nend] and the
    children of a node stored consecutively from first_child, in octant
    order.  Node 0 is the root."""
    pts = np.asarray(pts, dtype=float)
    n = pts.shape[0]
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    half = 0.5 * float((hi - lo).max()) + 1e-9
    perm = np.empty(n, dtype=np.int64)
    nbeg, nend, first, nch = [0], [0], [0], [0]
    fill = [0]

    def build(idx, center, half, depth, node):
        nbeg[node] = fill[0]
        if idx.size <= leaf_size or depth >= 48 or half < 1e-12:
            perm[fill[0]:fill[0] + idx.size] = idx
            fill[0] += idx.size
            nend[node] = fill[0]
            return
        sub = pts[idx]
        octant = ((sub[:, 0] > center[0]).astype(int) * 4
                  + (sub[:, 1] > center[1]).astype(int) * 2
                  + (sub[:, 2] > center[2]).astype(int))
        kids = [o for o in range(8) if np.any(octant == o)]
        base = len(nbeg)
        for _ in kids:
            nbeg.append(0)
            nend.append(0)
            first.append(0)
            nch.append(0)
        first[node], nch[node] = base, len(kids)
        for k, o in enumerate(kids):
            shift = (np.array([(o >> 2) & 1, (o >> 1) & 1, o & 1]) * 2.0 - 1.0) * (half / 2.0)
            build(idx[octant == o], center + shift, half / 2.0, depth + 1, base + k)
        nend[node] = fill[0]

    if n:
        build(np.arange(n), 0.5 * (lo + hi), half, 0, 0)
    return (perm, np.array(nbeg, dtype=np.int64), np.array(nend, dtype=np.int64),
            np.array(first, dtype=np.int64), np.array(nch, dtype=np.int32))


class TreePlan:
    """Device-resident topology + group index for one source geometry."""

    def __init__(self, sources, source_groups, leaf_size, device):
        import torch
        self.device = device
        perm, nbeg, nend, first, nch = build_topology(sources, leaf_size)
        i64 = dict(dtype=torch.int64, device=device)
        self.ns = sources.shape[0]
        self.nnodes = nbeg.size if self.ns else 0
        self.perm = torch.as_tensor(perm, **i64)
        self.src = torch.as_tensor(np.asarray(sources, dtype=float)[perm], dtype=torch.float64,
                                   device=device).contiguous()
        self.nbeg = torch.as_tensor(nbeg, **i64)
        self.nend = torch.as_tensor(nend, **i64)
        self.first = torch.as_tensor(first, **i64)
        self.nchild = torch.as_tensor(nch, dtype=torch.int32, device=device)
        g = np.asarray(source_groups, dtype=np.int64)
        valid = np.nonzero(g >= 0)[0]
        order = valid[np.argsort(g[valid], kind="stable")]
        self.ngroups = int(g.max()) + 1 if valid.size else 0
        gb = np.zeros(max(self.ngroups, 1), dtype=np.int64)
        ge = np.zeros(max(self.ngroups, 1), dtype=np.int64)
        if valid.size:
            gs = g[order]
            starts = np.searchsorted(gs, np.arange(self.ngroups), side="left")
            ends = np.searchsorted(gs, np.arange(self.ngroups), side="right")
            gb[:self.ngroups], ge[:self.ngroups] = starts, ends
        self.gorder = torch.as_tensor(order, **i64)
        self.gsrc = torch.as_tensor(np.asarray(sources, dtype=float)[order], dtype=torch.float64,
                                    device=device).contiguous()
        self.gbeg = torch.as_tensor(gb, **i64)
        self.gend = torch.as_tensor(ge, **i64)
        words = _native.load().sf_tree_work_doubles(self.nnodes)
        self.work = torch.empty(max(words, 1), dtype=torch.float64, device=device)

    def stokeslet(self, strengths, targets, target_groups, mu, theta, cell_tolerance, out=None):
        """(nt,3) device result for device strengths (ns,3) / targets (nt,3)."""
        import torch
        f = strengths.reshape(-1, 3)
        fp = f.index_select(0, self.perm).contiguous()
        gf = f.index_select(0, self.gorder).contiguous() if self.gorder.numel() else None
        if out is None:
            out = torch.empty((targets.shape[0], 3), dtype=torch.float64, device=self.device)
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _native.call("sf_tree_stokeslet", _ptr(targets), _ptr(target_groups), targets.shape[0],
                     _ptr(self.src), _ptr(fp), self.ns, _ptr(self.nbeg), _ptr(self.nend),
                     _ptr(self.first), _ptr(self.nchild), self.nnodes, _ptr(self.gsrc), _ptr(gf),
                     _ptr(self.gbeg), _ptr(self.gend), self.ngroups, float(theta),
                     float(cell_tolerance), float(mu), _ptr(self.work), _ptr(out), st)
        return out


def geometry_key(sources, source_groups, leaf_size):
    h = hashlib.blake2b(digest_size=16)
    h.update(np.ascontiguousarray(sources, dtype=float).tobytes())
    h.update(np.ascontiguousarray(source_groups, dtype=np.int64).tobytes())
    return (np.shape(sources), int(leaf_size), h.hexdigest())
