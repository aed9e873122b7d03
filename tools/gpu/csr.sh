python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "csr or uneven or multirank" 2>&1 | tail -4
