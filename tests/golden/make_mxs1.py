"""Write small MXS1 fixtures with the REAL reference writer (maxsim/streamio.py:57-88).

Run in the build container (the reference is importable only there):
    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mxs1.py
The fixtures (tests/golden/mxs1/*.mxs1) travel with the repo; the tests parse them with the
native reader, compare against the arrays saved next to them (mxs1_expected.npz), and check
that our writer reproduces them byte for byte (the streaming GPU tests then write their larger
corpora with our writer).
"""

import os

import numpy as np
from maxsim import DocBatch, EmbeddingMatrix, pack, quantize_per_token, write_embeddings
from maxsim.quant import QuantizedCorpus

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mxs1")


def main():
    os.makedirs(HERE, exist_ok=True)
    rng = np.random.default_rng(5)
    dense = rng.standard_normal((7, 9, 16)).astype(np.float32)
    write_embeddings(os.path.join(HERE, "dense_f32.mxs1"), DocBatch.from_dense(dense))
    write_embeddings(os.path.join(HERE, "dense_f16.mxs1"), DocBatch.from_dense(dense), elem="f16")
    lens = [3, 1, 8, 5, 2]
    docs = [EmbeddingMatrix(rng.standard_normal((n, 16)).astype(np.float32)) for n in lens]
    packed = pack(docs)
    write_embeddings(os.path.join(HERE, "packed_f32.mxs1"), packed)
    write_embeddings(os.path.join(HERE, "packed_f16.mxs1"), packed, elem="f16")
    qm = [quantize_per_token(EmbeddingMatrix(dense[b])) for b in range(dense.shape[0])]
    qc = QuantizedCorpus.from_matrices(qm)
    write_embeddings(os.path.join(HERE, "quant.mxs1"), qc)
    np.savez_compressed(os.path.join(HERE, "mxs1_expected.npz"), dense=dense, packed_tokens=packed.tokens,
                        packed_cu=packed.cu_seqlens, quant_q=qc.q, quant_scales=qc.scales)


if __name__ == "__main__":
    main()
