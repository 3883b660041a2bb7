# Convenience targets (the driver uses __graft_entry__.build()).
.PHONY: build test-cpu
build:
	python paper_2204_13393_b200/build.py --force
	python -c "import oracle; oracle.build(force=True)"
test-cpu:
	python -m pytest tests -x -q -m "not gpu"
