"""CPU oracle for the EP dispatch/combine path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package, and only as the checker or the timed
CPU reference.  The product (``paper_2512_19849_b200``) never imports it; the
product fails loudly when libepb200.so is missing.

Modules
-------
codec       TransferCmd / immediate-word codecs      (command.py, imm.py)
ring        SPSC batch push/pop over the ctl array    (kernels.py:23-104)
deliveries  receiver-side delivery application       (kernels.py:124-318)
ep          layout / dispatch / combine / LL / FP8

Pinning status:
* codec, ring, deliveries: pinned against golden vectors produced by running
  the reference itself (tests/golden/make_golden.py).
* ep.dispatch / ep.ll_dispatch routing order and dedup: pinned against the
  reference's apply_deliveries driven by a SPEC-faithful HT / LL delivery plan
  (tests/golden/*.npz), plus the SPEC.md examples.
* ep.combine / ep.ll_combine, ep.fp8_quant: the reference has NO executable
  code for these (SPEC.md:446-454 is prose; SPEC.md:475 calls FP8 out of
  scope), so they are pinned only to the SPEC's examples and to independent
  checks (torch's CPU e4m3 cast) — parity unpinned against reference code.
"""
