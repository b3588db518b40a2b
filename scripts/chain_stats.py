"""Column-chain statistics of the c3 plan for several chain cost settings (pcb_info)."""
import os, sys
sys.path.insert(0, ".")
from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.operator import ProductConvolutionOperator
inp = inputs.make_config("c3")
for env in [("0", "24", "0"), ("1", "8", "0"), ("1", "24", "0"), ("1", "60", "0"), ("1", "24", "1")]:
    os.environ["PCB_CHAINS"], os.environ["PCB_CHAIN_BETA"], os.environ["PCB_CHAIN_GROW"] = env
    op = ProductConvolutionOperator.from_inputs(inp, mode="local", max_batch=1)
    i = op.info
    print(env, "chains", i["n_column_chains"], "chained terms", i["n_chained_terms"], "groups", i["n_groups"],
          "rows_inv bytes/vec %.1f MB" % (i["kernel_bytes"]["rows_inv"] / 1e6), "cols flops/vec %.2f GF" % (i["kernel_flops"]["cols"] / 1e9))
