// ad2_group.h — internal interface of the host process group (ad2_group.cu) for ad2.cu.
#pragma once
#include <cstddef>

#include "../../include/ad2.h"

size_t ad2_group_type_size(int dtype);
// in-place sum of `count` elements of `buf` (host memory) over the group, in rank order; returns
// 0 on success (a failure or timeout is latched: ad2_group_failed)
int ad2_group_sum_host(ad2_group g, void* buf, size_t count, int dtype);
bool ad2_group_failed(ad2_group g);
int ad2_group_rank(ad2_group g);
int ad2_group_size(ad2_group g);
