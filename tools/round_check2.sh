#!/bin/bash
# Round-2 closing GPU session: full parity suite, smoke, the bench line (both arms).
o=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $o/rc2_pytest.log 2>&1; echo rc $? >> $o/rc2_pytest.log
timeout 300 python __graft_entry__.py smoke > $o/rc2_smoke.log 2>&1; echo rc $? >> $o/rc2_smoke.log
timeout 900 python bench.py > $o/rc2_bench.log 2>&1; echo rc $? >> $o/rc2_bench.log
timeout 600 python bench.py --impl reference > $o/rc2_bench_ref.log 2>&1; echo rc $? >> $o/rc2_bench_ref.log
