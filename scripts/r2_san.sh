#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash scripts/sanitize.sh
