mkdir -p gpurun_out
TC_SKINNY_WS=0 timeout 300 python tools/skinny_layouts.py
TC_SKINNY_WS=1 TC_SKINNY_WS_STAGES=6 timeout 300 python tools/skinny_layouts.py
