// Drop-in forwarder: the B200 engine replaces this reference header (include/kvclust_b200.hpp).
#pragma once
#include "kvclust_b200.hpp"
