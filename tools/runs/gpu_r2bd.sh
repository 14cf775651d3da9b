#!/bin/bash
# pinned H2D throughput of one C5 batch: one copy vs k concurrent chunks
timeout 300 python tools/h2d_probe.py > gpurun_out/r2bd_h2d.log 2>&1
