"""CPU oracle for the mmFHE hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import anything under ``oracle/``.  The product
path (``paper_2603_22437_b200``) never imports it and shares no code with it.

Parts:
  * ``ckks_ref.c`` + ``ckks.py`` -- O-RNS: plain RNS-CKKS, coefficient form,
    textbook NTT, '%'-based modular arithmetic, client side (keygen, encode,
    encrypt, decrypt) and the cloud evaluator ops;
  * ``bigint_ref.py`` -- O-BIG: Python big-int, tiny-N CKKS ring arithmetic
    used to pin O-RNS;
  * ``dsp.py`` -- O-DSP: the paper's closed forms in numpy float64;
  * ``circuits.py`` -- the mmFHE kernel circuits K1-K7, FC, chains, written
    over the O-RNS evaluator in the paper's order.
"""
