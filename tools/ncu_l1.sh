#!/bin/bash
# Targeted ncu metrics (L1 hit rate, L1->xbar request activity) for kernel variants.
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_requests_srcunit_tex_op_read.sum,launch__occupancy_limit_shared_mem,launch__shared_mem_config_size
mkdir -p gpurun_out
# CARVES="default 25": shared-memory carveouts to compare (default = the driver's)
for cv in ${CARVES:-default 25}; do
  if [ "$cv" != default ]; then export LW_WO_CARVEOUT=$cv; else unset LW_WO_CARVEOUT; fi
  echo "== carve=$cv"
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_wo_ -s 2 -c 1 python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | grep -E "^\s+(gpu__|l1tex|lts|sm__|launch)" 
done
unset LW_WO_CARVEOUT
echo "== micro"
timeout 300 ncu --metrics $M --clock-control none -k regex:k_gather python tools/micro/run_gather_bw.py 2>&1 | grep -E "k_gather|^\s+(gpu__|l1tex|lts|sm__|launch)"
