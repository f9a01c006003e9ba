"""CPU oracle for the batched denoising step — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_2605_29233_b200``) may import this
package.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, and only as the checker
(or the timed CPU baseline), never as the thing measured or shipped.

``bb_oracle`` is a float64 NumPy restatement of the reference's hot path
(``/root/reference/pkg/src/blockbatch/{model,decoding,scheduler}.py``),
extended with the LLaDA/Dream-shape architecture (RMSNorm, RoPE, GQA, SwiGLU)
that the reference does not have.  It is pinned against fixtures generated
from the reference itself (``tests/golden/make_golden.py``).
"""
