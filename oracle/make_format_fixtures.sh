#!/bin/sh
# Golden faith-model/v1 + faith-embedding/v1 files written by the UNMODIFIED reference
# (model::save_model / save_embedding via oracle/_ref/faith_cli_ref gen; build it with
# `make -C oracle compat`).  tests/test_formats.py loads them with paper_2209_12708_b200.formats
# and compares against gen_synthetic / gen_synthetic_input of the same seeds.
set -e
cd "$(dirname "$0")/.."
out=tests/golden/formats
mkdir -p $out
oracle/_ref/faith_cli_ref gen --layers 1 --heads 2 --embed 8 --ffn 16 --length 4 --act tanh --seed 5 \
  --model $out/m1.json --input-seed 6 --input $out/x1.json
oracle/_ref/faith_cli_ref gen --layers 2 --heads 4 --embed 16 --ffn 24 --length 6 --classes 3 --act silu --seed 9 \
  --model $out/m2.json --input-seed 10 --input $out/x2.json
oracle/_ref/faith_cli_ref verify --model $out/m1.json --input $out/x1.json --eps 0.01 --norm l2 > $out/m1_verify.txt
ls -l $out
