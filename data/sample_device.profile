# Synthetic 16-SM device used by the reference's tests and tutorial
# (values restated from the reference fixture; layout is this repo's own).
num_SM = 16
B_max = 8
W_max = 48
T_max = 1024
R_max = 65536
Z_max = 12288
freq_GHz = 1.3
mem_bandwidth_GBps = 144
mem_latency_cycles = 436
departure_del_coal_cycles = 4
departure_del_uncoal_cycles = 40
uncoal_per_mw = 32
load_bytes_per_warp = 128
issue_cycles = 4
