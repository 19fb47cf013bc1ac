timeout 600 python tools/tile_ab.py reddit 1 2 4 8
timeout 900 python tools/tile_ab.py powerlaw_gcn 1 4 16
