"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path (the
parity oracle and the CPU-baseline leg). Importable only from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference arm; the
product package paper_2507_03153_b200 never imports it."""
