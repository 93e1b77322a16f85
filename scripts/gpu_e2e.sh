for nb in 2 3 4 5; do for q in 1 0.8 0.6 0.45; do echo -n "bands=$nb taper=$q: "; DFG_HOST_STREAM=0 DFG_HOST_TAPER=$q DFG_HOST_BANDS=$nb ./scripts/host_probe 1024 1024 | grep filter_host; done; done
for nb in 2 3 4; do for q in 1 0.7; do echo -n "4096 bands=$nb taper=$q: "; DFG_HOST_STREAM=0 DFG_HOST_TAPER=$q DFG_HOST_BANDS=$nb ./scripts/host_probe 4096 4096 | grep filter_host; done; done
