#include "cpu_coattn.cpp"
extern int bench_main(int, char**);
int main(int argc, char** argv) { return bench_main(argc, argv); }
