python tools/host_bound.py c12
python tools/host_bound.py c5
python tools/host_bound.py c3
python tools/grid_one.py 8
python tools/grid_one.py 10
