"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 engine.

Nothing in `paper_1110_2561_b200/` imports this package.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and the
`--impl reference` arm) may use it, and only as the checker or as the
timed CPU reference — never as the product path.

Contents (each function cites the reference file:line it restates):

* `naive`      — explicit +/-1 spin arrays and a per-bond loop, the
                 restatement of /root/reference/pkg/src/isingdos/oracle.py,
                 generalised to free boundaries and per-bond signs.
* `port`       — the reference's vectorised numpy engine restated:
                 `_classify_batch` / `enumerate_shard` / `full_dos_timed`
                 (enumeration.py:167-235, 356-390) and `partition_point`
                 (thermo.py:37-88); the CPU baseline of bench.py.
* `enum_ref.c` — the same two formulations in plain C (naive per-bond and
                 bit-mask), multi-threaded, used to produce the N = 36
                 golden tables the reference cannot express (BASELINE
                 configs 3 and 4).  Built by `oracle/Makefile` into
                 `oracle/_ref/` (git-ignored).

Pinning: the restatements are checked in tests/test_oracle_pins.py against
fixtures produced by running the reference package itself
(tests/golden/make_reference_goldens.py) — the 4x4 80-cell table, the 5x5
table, the 3x3x4 table, odd shard slices, the rows=17 unaligned slice and
thermodynamics on seven lattices.  Free-boundary and +/-J lattices are not
expressible in the reference (lattice.py:83-85): for those
the oracle is pinned only by agreement of the two independent restatements
and by the invariants (sum 2^N, binomial marginals, flip symmetry), which
DESIGN.md records as "parity unpinned by the reference" for those lattices.
"""
