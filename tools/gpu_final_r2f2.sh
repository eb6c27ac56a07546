#!/bin/bash
# End of round 2f: full GPU suite and smoke at HEAD, then randomised parity sweeps of the pass, the
# streaming windows and the online hook against the oracle / the reference's loop.
set -u
O=gpurun_out/final_r2f2
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -1 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 500 python tools/fuzz_parity.py --what pass --seconds 420 --seed 21 > $O/fuzz_pass.log 2>&1; tail -1 $O/fuzz_pass.log
timeout 400 python tools/fuzz_parity.py --what stream --seconds 300 --seed 22 > $O/fuzz_stream.log 2>&1; tail -1 $O/fuzz_stream.log
timeout 300 python tools/fuzz_parity.py --what hook --seconds 200 --seed 23 > $O/fuzz_hook.log 2>&1; tail -1 $O/fuzz_hook.log
