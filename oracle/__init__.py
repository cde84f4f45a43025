"""CPU oracle for the nvrec recovery path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithm of the hot path
(arxiv 2604.27441 / ReVo, package ``nvrec`` plus the loss-mask construction
in ``rgbdstream``).  It exists to *check* the CUDA implementation and to
time the reference CPU path in ``bench.py --impl reference``; it is never
the thing measured or shipped.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import it.  The product package ``paper_2604_27441_b200`` never imports this
module and fails loudly when its CUDA library is missing.

Modules
-------
``nvrec_forward``  functional restatement of ``MaskedVideoModel.forward``
                   (reference ``pkg/nvrec/src/nvrec/model.py:82-122``) over a
                   plain state dict, in fp32 torch-CPU ops -- the same ATen
                   kernels the reference calls.
``recover``        restatement of ``RecoveryServer._recover``
                   (``pkg/nvrec/src/nvrec/server.py:181-196``) and its 16-bit
                   depth extension ``recover16`` (65535 in place of 255).
``lossmask``       restatement of the loss-mask construction:
                   ``Receiver._finalize_p`` zero-fill (``receiver.py:224-237``),
                   ``codec.parse_header``/``block_ranges``/``_corrupted_blocks``
                   /``decode`` mask assembly (``codec.py:159-201,250-320``) and
                   the wire bitset (``recovery.py:214-227``).
``codec``          ``codec.decode`` / ``decode_bytes`` zero-fill decode and
                   ``fec.rs_reconstruct`` (``codec.py:260-340``, ``fec.py:144-163``).
``baseline``       ``recover_baseline_rgb/_depth`` (``recovery.py:94-196``).
``metrics``        the SSIM of ``rgbdstream/metrics.py:41-72`` (north_star's
                   |dSSIM| <= 1e-3 bar).

Pinning
-------
The oracle is pinned against golden vectors produced by running the
UNMODIFIED reference in the build container (``tests/golden/make_golden.py``
imports ``/root/reference``); ``tests/test_oracle_golden.py`` checks the
model, ``_recover``, loss-mask (216 trials through the reference
``Receiver._finalize_p`` plus the ``codec.decode`` tail rule) and baseline
restatements, ``tests/test_codec_oracle.py`` the codec/RS restatement, and
``tests/test_ssim_oracle.py`` the SSIM metric restatement.
"""
