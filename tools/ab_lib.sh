#!/bin/bash
# A/B: time sdpa with the regular library and with an experimental build
python tools/clock_probe.py sdpa 2
cp paper_2507_11978_b200/_lib/libntb200.so /tmp/base.so
cp paper_2507_11978_b200/_lib/libntb200_exp.so paper_2507_11978_b200/_lib/libntb200.so
python tools/clock_probe.py sdpa 2
cp /tmp/base.so paper_2507_11978_b200/_lib/libntb200.so
