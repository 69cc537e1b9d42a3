DT=1 BX=32 SW=3 timeout 60 ./scripts/tma_probe 0 16 1 6
DT=1 BX=32 SW=0 timeout 60 ./scripts/tma_probe 0 16 1 6
BX=64 SW=3 timeout 60 ./scripts/tma_probe 0 16 1 6
BX=32 SW=0 timeout 60 ./scripts/tma_probe 0 32 32 0
