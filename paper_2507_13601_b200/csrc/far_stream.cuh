// far_stream.cuh — multi-batch concatenation kernels (§4).  (filled in below)
#pragma once
