// double instantiation of the launch sequences
#include "cmg_launch.cuh"
CMG_INSTANTIATE(double)
