"""oracle/ — TEST INFRASTRUCTURE ONLY (the checker, never the product).

CPU restatements of the reference algorithm for the pipelined load-and-use
path, used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  Nothing in paper_2210_16691_b200/ imports this.

- splitmix.py   : SplitMix64 + random_tensor (common.hpp:74-97, cli.hpp:41-46)
- alcop_oracle.c: C restatement (fp16/bf16 GEMM/BMM/conv with fp32
                  accumulation, pipeline index algebra, interpreter counters,
                  the reference analytical model) -> oracle/liboracle.so
- ref_driver.cpp: driver compiled from the reference headers themselves
                  (/root/reference, read-only) into oracle/_ref/ref_driver
"""
