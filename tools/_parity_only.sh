P=r02b; O=gpurun_out
python tools/parity_large.py c5 --out $O/${P}_parity_c5.json > $O/${P}_parity_c5.log 2>&1; echo "c5 rc=$?"
python tools/parity_large.py c4 --out $O/${P}_parity_c4.json > $O/${P}_parity_c4.log 2>&1; echo "c4 rc=$?"
python sweep.py --out $O/${P}_sweep_c4.jsonl > $O/${P}_sweep.log 2>&1; echo "sweep rc=$?"
python tools/fp32_edges.py > $O/${P}_fp32_edges.log 2>&1; tail -1 $O/${P}_fp32_edges.log
