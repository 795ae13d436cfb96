#!/bin/bash
# Regenerates the experiment-harness goldens from the REFERENCE's own
# sweep_batch_size / compare_policies (oracle/_ref/ref_experiment, built by
# `make -C oracle` from /root/reference/proj). Run where /root/reference exists.
#   fig13b_sweep.csv     sweep_batch_size over C = 16..256 (fig13b config, workload file)
#   fig14_compare.jsonl  compare_policies(intra_only -> rserve) over the fig14 config
set -e
cd "$(dirname "$0")"
make -s -C ../../oracle
tmp=$(mktemp -d)
../../oracle/_ref/ref_experiment fig13b_batch_size_32.json "$tmp/f13b" sweep 16,32,64,128,256
cp "$tmp/f13b/batch_size_sweep.csv" fig13b_sweep.csv
../../oracle/_ref/ref_experiment fig14_inter_ablation.json "$tmp/f14" compare intra_only rserve > fig14_compare.jsonl
rm -rf "$tmp"
