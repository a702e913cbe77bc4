#include <gtest/gtest.h>
int main() { return gt_run_all(); }
