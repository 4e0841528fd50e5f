timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_run.py --ligands 10000 --runs 1 | tail -1
python tools/batch_size.py
bash tools/gpu_quick.sh 2>&1 | grep "run 2"
