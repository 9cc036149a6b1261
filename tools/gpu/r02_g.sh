#!/bin/bash
# 4-GPU box: graphed DDP baseline (fixed capture), VGG-19 bs8 link-channel variants,
# ResNet-101 1 MB buckets with / without one-shot, GPT-2 lines.
mkdir -p gpurun_out
R=tools/gpu/recipes.sh
$R bench r02g_ddpgraph_r101_n4 4 --impl ddp --ddp-graphs
$R bench r02g_ddpgraph_vgg19_b8_n4 4 --impl ddp --ddp-graphs --model vgg19 --batch 8
$R bench r02g_vgg19_b8_n4 4 --model vgg19 --batch 8 --no-cpu-baseline
$R bench r02g_vgg19_b8_n4_sm 4 --model vgg19 --batch 8 --no-cpu-baseline --links sm
$R bench r02g_vgg19_b8_n4_ce 4 --model vgg19 --batch 8 --no-cpu-baseline --links ce
$R bench r02g_r101_1mb_n4 4 --bucket-mb 1 --no-cpu-baseline
$R bench r02g_r101_1mb_os1_n4 4 --bucket-mb 1 --oneshot-mb 1 --no-cpu-baseline
$R bench r02g_gpt2_n4 4 --model gpt2 --no-cpu-baseline
$R bench r02g_ddpgraph_gpt2_n4 4 --impl ddp --ddp-graphs --model gpt2
$R bench r02g_vgg19_n4 4 --model vgg19 --no-cpu-baseline
$R bench r02g_ddpgraph_vgg19_n4 4 --impl ddp --ddp-graphs --model vgg19
