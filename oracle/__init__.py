"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the page-update path.

Nothing in ``paper_2303_02868_b200`` imports this package.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its CPU-baseline
leg and ``--impl reference``) may use it, and only as the checker or as the
timed reference arm — never as the product path.

Contents
  page_adam.py   numpy restatement of hiermem/lockfree.py:127-263
                 (apply_update, MasterState.update_layer, ParamBuffer
                 accumulate/take/publish) plus exact bf16 RNE, page pack /
                 unpack over (page, offset, bytes) segments.
  gen_golden.py  writes tests/golden/* by calling the reference package
                 itself (/root/reference/pkg/src, this container only).

Parity pinning: tests/test_oracle.py checks page_adam.py bit-for-bit
against tests/golden/adam_golden.npz, which gen_golden.py produced by
running the reference's own ``apply_update`` / ``MasterState`` /
``ParamBuffer`` on seeded inputs.  The page table (csrc/pagetable.cpp) is
pinned directly against reference ``state_dict`` dumps in
tests/golden/pagetable_*.json.gz.
"""
