#!/bin/bash
# quick box facts for DESIGN.md / bench sizing
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv; lscpu | grep -E "Model name|Socket|Thread|Core" 
