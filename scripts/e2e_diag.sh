# e2e leg diagnostics on whatever box this lands on: raw pinned copy rates,
# the e2e probe's phase split, and the bench's own e2e leg
mkdir -p gpurun_out
{
python scripts/pcie_probe.py
PYTHONPATH=$PWD python scripts/e2e_probe.py
echo "bench e2e $(timeout 300 python bench.py --no-cpu --no-config2 --no-aggregate 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["ms_per_step"])')"
nvidia-smi -q | grep -i -A3 "Link Width\|PCIe Generation" | head -20
} > gpurun_out/e2e_diag_$(date +%s).log 2>&1
