echo default; timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
echo pull2; IMX_HOOK=pull IMX_PULL_HEAVY=2 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
echo hybrid3; IMX_HOOK=hybrid IMX_PULL_HEAVY=3 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
echo pull1; IMX_HOOK=pull IMX_PULL_HEAVY=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()"
