"""CPU restatement of the reference algorithm — TEST INFRASTRUCTURE ONLY.

This package is the parity *checker* for the B200 path, never part of it.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
package ``paper_2512_02371_b200`` never imports it and has no CPU fallback.

Modules
  interp_ref     restated interpreter semantics of the hot path
                 (/root/reference/pkg/src/tensorsel/interp.py): rounding,
                 SplitMix64 fills, wmma tile gathers, left-to-right f32
                 contraction, the source-form conv statement.
  layout_ref     restated Toeplitz-family builders (layout.py), loop form.
  pipelines_ref  image-level pipelines composed from the two above:
                 separable Lanczos-3 resample, Gaussian/box filters, DCT-16
                 denoise (§V-C/E), clamp-to-edge.

Pinning.  Tile-level semantics (rounding, generators, window x matrix,
conv/downsample/upsample statements, accumulation order) are pinned
bit-exactly to the reference by the fixtures in tests/golden/, produced by
oracle/make_golden.py from the reference itself (interp.run_program on the
corpus and on generated Lanczos / Gaussian tile programs).  The image-level
composition (separable order, clamp policy, Lanczos/Gaussian/box weights,
DCT denoise) has no reference code: it is restated from PAPER.md and is
"parity unpinned" beyond the 1-D row pass it is built from.
"""
