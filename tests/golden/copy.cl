__kernel void copy(__global int *data, int x) {
    data[get_global_id(0) - get_global_offset(0)] = x;
}
