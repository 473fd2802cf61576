"""numpy stand-in for the CUDA store's shard-engine interface (TEST INFRASTRUCTURE).

Lets ``paper_2504_18943_b200.dist`` -- the multi-GPU exchange protocol -- run under gloo on
CPU.  It enumerates a level's candidates with plain numpy lane arithmetic (written
independently of both the CUDA kernels and the C oracle), takes the ordinals that belong to
its shard, keeps ``{CM bytes -> min ordinal}`` for CMs not stored at an earlier level, and
finalises by sorting winners by ordinal.  The tests compare the levels it ends up with, on
every rank, with the C oracle's (``oracle/``), which pins the protocol end to end.
"""

from __future__ import annotations

import zlib

import numpy as np
import torch

from paper_2504_18943_b200.engine import OP_AND, OP_ATOM, OP_FUTURE, OP_NEXT, OP_NOT, OP_OR, OP_UNTIL
from paper_2504_18943_b200.traces import Layout, atom_bitvectors, smallest_lane_dtype

NO_SEPARATOR = (1 << 64) - 1


class _Level:
    def __init__(self, cms, op, left, right, base):
        self.cms, self.op, self.left, self.right, self.base = cms, op, left, right, base

    @property
    def n(self):
        return len(self.cms)


class CpuShardEngine:
    def __init__(self, spec):
        self.spec = spec
        self.dtype = smallest_lane_dtype(spec.max_length)
        self.layout = Layout.from_specification(spec, self.dtype)
        self.atoms = np.array(atom_bitvectors(spec, self.dtype))
        self.T = spec.trace_count
        self.row_bytes = self.T * self.dtype.itemsize
        self.key_bytes = -(-self.row_bytes // 16) * 16
        self.levels: list[_Level] = []
        self.seen: set[bytes] = set()
        self.has_separator = False
        self.torch_device = torch.device("cpu")
        self._pending = None

    @property
    def total(self):
        return sum(lv.n for lv in self.levels)

    def level(self, cost):
        return self.levels[cost - 1]

    def entry(self, gid):
        for lv in self.levels:
            if lv.base <= gid < lv.base + lv.n:
                k = gid - lv.base
                return int(lv.op[k]), int(lv.left[k]), int(lv.right[k])
        raise IndexError(gid)

    # ---- lane arithmetic (numpy, one array element per trace lane) -----------------------
    def _shifts(self):
        w, s, out = self.dtype.itemsize * 8, 1, []
        while s < w:
            out.append(s)
            s *= 2
        return out

    def _apply(self, op, a, b=None):
        one = self.dtype.type
        if op == OP_NOT:
            return (~a) & self.layout.masks
        if op == OP_NEXT:
            return a >> one(1)
        if op == OP_FUTURE:
            x = a.copy()
            for s in self._shifts():
                x |= x >> one(s)
            return x
        if op == OP_AND:
            return a & b
        if op == OP_OR:
            return a | b
        r, q = b.copy(), a.copy()
        for s in self._shifts():
            r |= q & (r >> one(s))
            q &= q >> one(s)
        return r & self.layout.masks

    # ---- canonical block list of a level --------------------------------------------------
    def _blocks(self, cost, op_mask):
        blocks, ord0 = [], 0

        def add(op, kind, la, lb):
            nonlocal ord0
            na = la.n if la is not None else self.atoms.shape[0]
            nb = lb.n if lb is not None else 0
            size = na if kind == "unary" else (na * (na + 1) // 2 if kind == "tri" else na * nb)
            if size:
                blocks.append(dict(op=op, kind=kind, la=la, lb=lb, na=na, nb=nb, ord0=ord0, size=size))
                ord0 += size

        if cost == 1:
            add(OP_ATOM, "unary", None, None)
            return blocks, ord0
        prev = self.levels[cost - 2]
        for op in (OP_NOT, OP_NEXT, OP_FUTURE):
            if op_mask >> op & 1 and prev.n:
                add(op, "unary", prev, None)
        for op in (OP_AND, OP_UNTIL, OP_OR):
            if not op_mask >> op & 1:
                continue
            commutative = op in (OP_AND, OP_OR)
            for c1 in range(1, cost - 1):
                c2 = cost - 1 - c1
                if commutative and c1 > c2:
                    break
                la, lb = self.levels[c1 - 1], self.levels[c2 - 1]
                if la.n == 0 or lb.n == 0:
                    continue
                add(op, "tri" if commutative and c1 == c2 else "rect", la, lb)
        return blocks, ord0

    @staticmethod
    def _pairs(block, local):
        """(i, j) of block-local ordinals (numpy int64 arrays)."""
        if block["kind"] == "unary":
            return local, None
        if block["kind"] == "rect":
            return local // block["nb"], local % block["nb"]
        n = block["na"]
        starts = np.array([i * n - (i * (i - 1)) // 2 for i in range(n)], dtype=np.int64)
        i = np.searchsorted(starts, local, side="right") - 1
        return i, i + (local - starts[i])

    def _decode(self, blocks, ords):
        starts = np.array([b["ord0"] for b in blocks], dtype=np.int64)
        which = np.searchsorted(starts, ords, side="right") - 1
        op = np.empty(len(ords), dtype=np.uint8)
        left = np.empty(len(ords), dtype=np.int64)
        right = np.full(len(ords), -1, dtype=np.int64)
        for bi, b in enumerate(blocks):
            sel = np.flatnonzero(which == bi)
            if not len(sel):
                continue
            i, j = self._pairs(b, ords[sel] - b["ord0"])
            op[sel] = b["op"]
            left[sel] = i if b["la"] is None else b["la"].base + i
            if j is not None:
                right[sel] = (b["la"] if b["kind"] == "tri" else b["lb"]).base + j
        return op, left, right

    def _key(self, row) -> bytes:
        return row.tobytes().ljust(self.key_bytes, b"\0")

    # ---- shard-engine interface (paper_2504_18943_b200.dist.ShardEngine) -------------------------------------
    def _enumerate(self, cost, op_mask, shard_index, shard_count):
        """(blocks, constructed, candidate rows, ordinals) of this shard: ordinals strided over the ranks."""
        blocks, constructed = self._blocks(cost, op_mask)
        rows, ords = [], []
        for b in blocks:
            local = np.arange(b["size"], dtype=np.int64)
            local = local[(b["ord0"] + local) % shard_count == shard_index]
            if not len(local):
                continue
            i, j = self._pairs(b, local)
            if b["kind"] == "unary":
                src = self.atoms if b["la"] is None else b["la"].cms
                cand = src[i] if b["op"] == OP_ATOM else self._apply(b["op"], src[i])
            else:
                lb = b["la"] if b["kind"] == "tri" else b["lb"]
                cand = self._apply(b["op"], b["la"].cms[i], lb.cms[j])
            rows.append(cand)
            ords.append(b["ord0"] + local)
        if rows:
            return blocks, constructed, np.concatenate(rows), np.concatenate(ords)
        return blocks, constructed, np.empty((0, self.T), dtype=self.dtype), np.empty(0, dtype=np.int64)

    def _owner(self, key: bytes, owners: int) -> int:
        return zlib.crc32(key) % owners

    def _records(self, items):
        """(rows uint8 [n, key_bytes], ords int64 [n]) tensors of (key, ordinal) pairs."""
        rows = np.frombuffer(b"".join(k for k, _ in items), dtype=np.uint8).reshape(len(items), self.key_bytes).copy() \
            if items else np.empty((0, self.key_bytes), dtype=np.uint8)
        return torch.from_numpy(rows), torch.from_numpy(np.array([o for _, o in items], dtype=np.int64))

    def route_begin(self, cost, op_mask, exhaustive, deadline, rank, world):
        blocks, constructed, cand, ords = self._enumerate(cost, op_mask, rank, world)
        sep_flags = ((cand & self.dtype.type(1)) == self.layout.target).all(axis=1) if len(cand) else np.zeros(0, bool)
        seps = [int(o) for o in ords[sep_flags]]
        # while the store holds no separating CM, a separating candidate cannot repeat an older CM
        sep_local = min(seps) if seps and not self.has_separator else NO_SEPARATOR
        per_owner = [[] for _ in range(world)]
        for k in range(len(ords)):
            key = self._key(cand[k])
            per_owner[self._owner(key, world)].append((key, int(ords[k])))
        self._pending = dict(cost=cost, blocks=blocks, constructed=constructed, seps=seps, exhaustive=exhaustive,
                             rank=rank, world=world, claims={}, recv=None, bitmap=None)
        return 0, [self._records(items) for items in per_owner], sep_local, len(seps)

    def exchange_recv(self, n_records):
        rows = torch.empty((n_records, self.key_bytes), dtype=torch.uint8)
        ords = torch.empty((n_records,), dtype=torch.int64)
        self._pending["recv"] = (rows, ords)
        return rows, ords

    def owner_reduce(self, n_records):
        p = self._pending
        rows, ords = p["recv"]
        raw, claims = rows.numpy(), p["claims"]
        for k in range(n_records):
            key, o = raw[k].tobytes(), int(ords[k])
            assert self._owner(key, p["world"]) == p["rank"], "a record reached a rank that does not own it"
            if key not in self.seen and o < claims.get(key, NO_SEPARATOR):
                claims[key] = o
        words = np.zeros((p["constructed"] + 31) // 32 + 1, dtype=np.uint32)
        for o in claims.values():
            words[o >> 5] |= np.uint32(1 << (o & 31))
        p["bitmap"] = torch.from_numpy(words.view(np.int32))
        return 0, p["bitmap"]

    def winners_export(self, sep_ord):
        p = self._pending
        cut = (not p["exhaustive"]) and sep_ord != NO_SEPARATOR
        p["winners"] = [(k, o) for k, o in p["claims"].items() if not cut or o <= sep_ord]
        return self._records(p["winners"])

    def level_abort(self):
        if self._pending is not None:
            self.levels.append(_Level(np.empty((0, self.T), dtype=self.dtype), np.empty(0, np.uint8), np.empty(0, np.int64),
                                      np.empty(0, np.int64), self.total))
            self._pending = None

    def separating_ordinals(self):
        return torch.tensor(self._pending["seps"], dtype=torch.int64)

    def level_commit(self, sep_ord, seps, recv_counts, batch_size, memory_budget_bytes):
        p = self._pending
        n_received = sum(recv_counts)
        rows, ords = p["recv"] if n_received else (None, None)
        items = [(o, k) for k, o in p["winners"]]
        for k in range(n_received):
            items.append((int(ords[k]), rows[k].numpy().tobytes()))
        items.sort()
        # the all-reduced bitmap is the level's winners: one bit per entry, at its ordinal
        bits = p["bitmap"].numpy().view(np.uint32)
        cut = (not p["exhaustive"]) and sep_ord != NO_SEPARATOR
        marked = [o for o in np.flatnonzero(np.unpackbits(bits.view(np.uint8), bitorder="little")) if not cut or o <= sep_ord]
        assert marked == [o for o, _ in items], "winners bitmap and published winners disagree"
        if sep_ord != NO_SEPARATOR or (seps is not None and len(seps)):
            self.has_separator = True
        return self._append(p, items, sep_ord)

    def _append(self, p, items, sep_ord):
        ords = np.array([o for o, _ in items], dtype=np.int64)
        base = self.total
        if items:
            cms = np.frombuffer(b"".join(k[: self.row_bytes] for _, k in items), dtype=self.dtype).reshape(len(items), self.T).copy()
            op, left, right = self._decode(p["blocks"], ords)
        else:
            cms = np.empty((0, self.T), dtype=self.dtype)
            op, left, right = np.empty(0, np.uint8), np.empty(0, np.int64), np.empty(0, np.int64)
        for _, k in items:
            self.seen.add(k)
        self.levels.append(_Level(cms, op, left, right, base))
        sep_gid = None
        if sep_ord != NO_SEPARATOR:
            pos = int(np.searchsorted(ords, sep_ord))
            if pos < len(ords) and ords[pos] == sep_ord:
                sep_gid = base + pos
        self._pending = None
        return 0, len(items), sep_gid, p["constructed"]

    def level_candidates(self, cost, op_mask):
        return self._blocks(cost, op_mask)[1]

    def expand_local(self, cost, op_mask, exhaustive, batch_size, memory_budget_bytes, deadline):
        """The whole level on this rank: what dist.py does for levels below REPLICATE_BELOW."""
        blocks, constructed, cand, ords = self._enumerate(cost, op_mask, 0, 1)
        claims: dict[bytes, int] = {}
        sep_flags = ((cand & self.dtype.type(1)) == self.layout.target).all(axis=1) if len(cand) else np.zeros(0, bool)
        sep_ord = NO_SEPARATOR
        for k in range(len(ords)):
            key, o = self._key(cand[k]), int(ords[k])
            fresh = key not in self.seen
            if fresh and o < claims.get(key, NO_SEPARATOR):
                claims[key] = o
            if sep_flags[k]:
                self.has_separator = True
                if fresh:
                    sep_ord = min(sep_ord, o)
        cut = (not exhaustive) and sep_ord != NO_SEPARATOR
        items = sorted((o, k) for k, o in claims.items() if not cut or o <= sep_ord)
        return self._append(dict(blocks=blocks, constructed=constructed), items, sep_ord)
