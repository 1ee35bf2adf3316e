# NVIDIA B200 (sm_100a) device profile in the reference's profile format.
# Occupancy limits are the architectural per-SM limits; timing constants are
# documented ASSUMPTIONS (microbenchmarking is outside the reference's scope),
# chosen from this repo's measurements where one exists:
#   mem_bandwidth_GBps = MEASURED_PEAKS.json hbm_gbs (6552.3 GB/s copy),
#   freq_GHz = clocks.max.sm 1965 MHz.
R_max = 65536            # 64K 32-bit registers per SM
Z_max = 58368            # 228 KB shared memory per SM, in 4-byte words
T_max = 1024
B_max = 32
W_max = 64
num_SM = 148
freq_GHz = 1.965
mem_latency_cycles = 600
departure_del_coal_cycles = 4
departure_del_uncoal_cycles = 40
mem_bandwidth_GBps = 6552.3
issue_cycles = 4
load_bytes_per_warp = 128
uncoal_per_mw = 32
