"""CPU oracle for arXiv 1905.05233 (Winograd convolution beyond linear polynomials).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
``paper_1905_05233_b200``, its C-ABI library ``libwino.so`` and its CUDA
kernels) may import, call, link or execute anything under ``oracle/``.  The only
permitted users are ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.

The oracle is a plain, slow, obviously-correct restatement of the paper:

* ``exact``      -- polynomials over Q.
* ``transforms`` -- Toom-Cook sub-solver, Algorithm 1 (G^W, A^W), Algorithm 2
                    (B^W = [EC | vec M]), role assignment of Eq. (2), the
                    multiplication count / ratio of Sec. 2.3, and the residue-block
                    matrices used by the "2x2-block product mod m_i" lowering.
* ``conv``       -- direct (valid) correlation in fp64 and exact-rational Winograd
                    (1D, 2D single tile, tiled multi-channel layer).
* ``precision``  -- rounding primitives and the two emulated-precision models:
                    PAPER mode (every scalar op in fp32 then cast down) and
                    PIPELINE mode (rounding only at stored tensors V, U, y).
* ``metrics``    -- error statistics (SURVEY.md 8(b) stats layout).

Every function cites the passage it follows.  Parity status of each function is
listed in DESIGN.md ("Oracle pins").  Functions whose *absolute* output values
have no independent pin say "parity unpinned" in their docstring: these are the
absolute error magnitudes of the emulated-precision models (Figure 1 of the
paper is missing from PAPER.md); their *trends* are pinned.
"""
