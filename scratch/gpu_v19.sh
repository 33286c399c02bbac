timeout 900 python -m pytest tests -m gpu -x -q -k "lookup or multiplicities or pair" 2>&1 | tail -2
python scratch/cfg3_prof.py 2>&1 | head -8
