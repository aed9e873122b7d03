python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/probe_e2e.py c2 explicit
python tools/probe_e2e.py c2 gram
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
