"""pareto_sweep host side: row schema and table format pinned to the
reference (simulator.py:997-998, 1047-1055).  The expected table below was
printed by the reference's own ``pareto_to_table`` on these rows
(PYTHONPATH=/root/reference/pkg/src python -c 'from burstplan.simulator
import pareto_to_table; ...')."""

import paper_2112_10065_b200 as bpx
from paper_2112_10065_b200.sweep import PARETO_HEADER, pareto_to_table

ROWS = [
    {"label": "bp+col amp=2 pace=2 bg=8", "scenario": "bp+col", "amp_limit": 2.0,
     "fg_speedup": 1.23456789, "fg_iteration_us": 15552.95715,
     "cluster_throughput": 4484.8372101, "bg_throughput": 2480.44069},
    {"label": "partition k=1", "scenario": "partition", "amp_limit": float("nan"),
     "fg_speedup": 1.0, "fg_iteration_us": 15600.0, "cluster_throughput": 2051.28205,
     "bg_throughput": 0.0},
]
REF_TABLE = ("label\tscenario\tamp_limit\tfg_speedup\tfg_iteration_us\tcluster_throughput"
             "\tbg_throughput\nbp+col amp=2 pace=2 bg=8\tbp+col\t2\t1.2346\t15552.957\t"
             "4484.837\t2480.441\npartition k=1\tpartition\tnan\t1.0000\t15600.000\t"
             "2051.282\t0.000\n")


def test_header_matches_reference():
    assert PARETO_HEADER == ("label", "scenario", "amp_limit", "fg_speedup",
                             "fg_iteration_us", "cluster_throughput", "bg_throughput")
    assert bpx.PARETO_HEADER is PARETO_HEADER


def test_table_matches_reference_bytes():
    assert pareto_to_table(ROWS) == REF_TABLE


def test_exported_lazily():
    assert callable(bpx.pareto_sweep) and callable(bpx.pareto_to_table)
