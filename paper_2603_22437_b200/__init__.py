"""B200-native (sm_100a) mmFHE cloud-side hot path: RNS-CKKS evaluation of the
mmFHE kernel chains (arxiv 2603.22437) behind the C-ABI of include/mmfhe.h.

    from paper_2603_22437_b200 import mmfhe
    ctx = mmfhe.Context.from_params(params, device=0)

The CUDA library is ``lib/libmmfhe.so`` (built by ``python -m
paper_2603_22437_b200.build``); there is no CPU fallback.
"""
