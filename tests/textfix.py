"""Text fixtures -> token ids.  Test-side only: the generator
works in the token-id domain, so tokenization is not on the GPU path."""
import string

import numpy as np

from workload.gen import PH, VOCAB_BASE

PUNCT = set(string.punctuation)


def fragments(text: str):
    out = []
    for w in text.split():
        if w == "<*>":
            out.append(w)
            continue
        lead, trail = [], []
        while w and w[0] in PUNCT:
            lead.append(w[0]); w = w[1:]
        while w and w[-1] in PUNCT:
            trail.insert(0, w[-1]); w = w[:-1]
        out.extend(lead + ([w] if w else []) + trail)
    return out


class Interner:
    def __init__(self):
        self.ids = {}

    def __call__(self, text: str) -> np.ndarray:
        toks = []
        for f in fragments(text):
            if f == "<*>":
                toks.append(PH)
                continue
            if f not in self.ids:
                self.ids[f] = VOCAB_BASE + len(self.ids)
            toks.append(self.ids[f])
        return np.array(toks, dtype=np.uint32)


def pool_from_demos(demos, interner):
    """demos: list of {log, template} -> workload.gen.Pool (template ids by first appearance)."""
    from workload.gen import Pool
    logs = [interner(d["log"]) for d in demos]
    tpls = [interner(d["template"]) for d in demos]
    tid, tids = {}, []
    for d in demos:
        tids.append(tid.setdefault(d["template"], len(tid)))
    lo = np.concatenate([[0], np.cumsum([len(x) for x in logs])]).astype(np.uint32)
    to = np.concatenate([[0], np.cumsum([len(x) for x in tpls])]).astype(np.uint32)
    return Pool(lo, np.concatenate(logs).astype(np.uint32), to, np.concatenate(tpls).astype(np.uint32),
                np.array(tids, np.uint32), np.arange(len(demos), dtype=np.uint32))
