#!/bin/bash
# sample SM clocks / power / throttle reasons every 200 ms into $1 until killed
while true; do nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> "$1"; sleep 0.2; done
