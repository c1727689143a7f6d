"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference ``kkbeam`` hot path (see
``kkbeam_oracle.py`` and ``kk_oracle.c``).  Importable only from ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline arm, as the
checker; the product package ``paper_2603_22496_b200`` never imports it.
"""
