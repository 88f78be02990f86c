"""A host (numpy/torch-CPU) stand-in for the column-keyed CUDA generator of
paper_1911_07722_b200.configs (csrc/datagen.cu), used only by the CPU tests
of the shard-local data path.  Same contract -- every value is a function of
(seed, tag, global column or id) -- different streams (numpy's Philox)."""
import numpy as np
import torch


class HostGen:
    def __init__(self, seed=0):
        self.seed = seed

    def _gen(self, tag, col):
        return np.random.Generator(np.random.Philox(key=[self.seed, tag],
                                                    counter=[0, int(col), 0, 0]))

    @staticmethod
    def _list(ids):
        return list(range(ids)) if isinstance(ids, int) else [int(x) for x in ids]

    def normal_cols(self, ids, d, lda):
        cols = self._list(ids)
        out = np.zeros((len(cols), lda), dtype=np.float32)
        for s, j in enumerate(cols):
            out[s, :d] = self._gen(1, j).standard_normal(d, dtype=np.float32)
        return torch.from_numpy(out)

    def ids(self, ids, tag, uniform=False):
        idl = self._list(ids)
        g = self._gen(100 + tag, 0)
        # one value per id from one keyed stream: draw up to max id, index
        top = (max(idl) + 1) if idl else 0
        vals = g.random(top) if uniform else g.standard_normal(top)
        return torch.from_numpy(vals[idl] if idl else np.zeros(0))

    def onehot(self, ids, d, nnz, cdf):
        cols = self._list(ids)
        c = cdf.numpy()
        out = np.zeros((len(cols), nnz), dtype=np.int32)
        for s, j in enumerate(cols):
            g = self._gen(6, j)
            got = []
            while len(got) < nnz:
                f = int(min(np.searchsorted(c, g.random()), d - 1))
                if f not in got:
                    got.append(f)
            out[s] = np.sort(got)
        return torch.from_numpy(out)
