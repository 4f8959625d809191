#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout -k 10 1500 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
