"""Flat model of the sibling/version protocol.  TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

Restates /root/reference/pkg/src/hetrt/memory.py:118-227 literally over a
dict (area, space) -> [version, valid, bytes|None] with no handles, in the
spirit of the reference's own brute-force model (tests/refmodel.py:13-94):
request-read copies the max-version valid sibling (host first, else lowest
space id) unless resident; protect backs up a sole max-version copy that
lives in the attempt's (non-host) space to the host; writes return a token
(area, space, top+1, buffer) that commit applies; rollback invalidates.
"""

from __future__ import annotations


class ModelDataLoss(Exception):
    pass


class SiblingModel:
    def __init__(self, host: str = "host"):
        self.host = host
        self.t: dict = {}
        self.size: dict = {}
        self.n = 0

    def register(self, payload: bytes) -> str:
        a = f"a{self.n}"
        self.n += 1
        self.size[a] = len(payload)
        self.t[(a, self.host)] = [0, True, bytes(payload)]
        return a

    def _newest(self, a):
        live = {sp: e for (x, sp), e in self.t.items() if x == a and e[1]}
        if not live:
            raise ModelDataLoss(a)
        top = max(e[0] for e in live.values())
        return top, {sp: e for sp, e in live.items() if e[0] == top}

    def _src(self, newest):
        return newest[self.host] if self.host in newest else newest[min(newest)]

    def _backup(self, a, space, protect):
        if not protect or space == self.host:
            return
        top, newest = self._newest(a)
        if set(newest) == {space}:
            self.t[(a, self.host)] = [top, True, bytes(newest[space][2])]

    def read(self, a, space, protect=False):
        top, newest = self._newest(a)
        e = self.t.get((a, space))
        if e is None or not e[1] or e[0] != top:
            self.t[(a, space)] = [top, True, bytes(self._src(newest)[2])]
        self._backup(a, space, protect)
        e = self.t[(a, space)]
        return e[0], bytes(e[2])

    def write(self, a, space, access, protect=False):
        top, newest = self._newest(a)
        self._backup(a, space, protect)
        if access == "rw":
            e = self.t.get((a, space))
            buf = bytearray(e[2]) if (e is not None and e[1] and e[0] == top) else bytearray(self._src(newest)[2])
        else:
            buf = bytearray(self.size[a])
        self.t.setdefault((a, space), [top, False, None])
        return [a, space, top + 1, buf]

    def commit(self, tok):
        a, space, ver, buf = tok
        self.t[(a, space)] = [ver, True, bytes(buf)]

    def invalidate(self, a, space):
        self.t[(a, space)][1] = False

    def rollback(self, areas, space):
        if space == self.host:
            return
        for a in areas:
            if (a, space) in self.t:
                self.t[(a, space)][1] = False
