"""ORACLE — test infrastructure only.

CPU restatements of the reference (`/root/reference/pkg/src/ddschur`) used
as the parity checker by `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py`.  Nothing in the
product package (`paper_2203_10879_b200/`) imports this package.
"""
